"""ncu launch list (--metrics gpu__time_duration.sum --csv) -> markdown table of kernels by total time.

    python tools/launches_md.py gpurun_out/launches.csv "<command>" "<note>" > profiles/rNN/launches_x.md
"""
import collections
import csv
import sys


def main(path, cmd="", note=""):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki][:90]
        tot[name] += float(r[vi].replace(",", "")) / 1e3
        cnt[name] += 1
    total = sum(tot.values())
    print(f"# ncu launch list of `{cmd}`\n")
    print("Cold-cache, serialised (ncu --metrics gpu__time_duration.sum --clock-control none): compare shares, not absolutes.")
    if note:
        print(note)
    print("\n| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{name}` | {cnt[name]} | {t:.1f} | {t / cnt[name]:.1f} | {t / total:.3f} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
