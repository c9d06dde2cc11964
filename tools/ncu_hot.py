"""Top SASS instructions by warp-stall samples from an ncu report (run here, on the CPU box).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(path, n=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    data = [(int(r[i_s] or 0), r[hdr.index("Address")], r[i_src].strip()) for r in rows[2:] if len(r) > i_s]
    tot = sum(d[0] for d in data) or 1
    kinds = {}
    for s, _, src in data:
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        kinds[op.split(".")[0]] = kinds.get(op.split(".")[0], 0) + s
    print("stall samples by opcode:", sorted(((round(100 * v / tot, 1), k) for k, v in kinds.items()), reverse=True)[:12])
    for s, a, src in sorted(data, reverse=True)[:n]:
        print(f"{100 * s / tot:5.1f}%  {a}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
