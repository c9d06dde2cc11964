"""Turn suite JSON lines (tools/suite.py) into the markdown table committed under profiles/."""
import json
import sys


def fmt(x, spec=".3g"):
    return "—" if x is None else format(x, spec)


def main(path):
    rows = []
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "error" in d:
            rows.append(f"| error | {' '.join(d.get('cmd', []))} | | | | | | |")
            continue
        r = d.get("roofline") or {}
        cpu = d.get("cpu_baseline") or {}
        e2e = d.get("e2e") or {}
        ratio = (d["value"] / cpu["value"]) if cpu.get("value") else None
        rows.append(
            f"| {d['config']['workload']} | {d['dtype']} | {fmt(d['value'])} | {fmt(r.get('achieved'), '.0f')} | "
            f"{fmt(r.get('frac'), '.3f')} | {fmt(r.get('kernel_avg_ms'), '.4f')} | {fmt(e2e.get('value'))} | "
            f"{fmt(cpu.get('value'))} ({cpu.get('cores', '—')} core) | {fmt(ratio, '.3g')} |"
        )
    print("| workload | dtype | GPU site-ops/s | kernel GB/s (algorithmic) | of measured HBM | kernel ms | e2e site-ops/s | CPU reference port site-ops/s | GPU/CPU |")
    print("|---|---|---|---|---|---|---|---|---|")
    print("\n".join(rows))


if __name__ == "__main__":
    main(sys.argv[1])
