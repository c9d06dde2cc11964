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
        par = d.get("parity") or {}
        ratio = (d["value"] / cpu["value"]) if cpu.get("value") else None
        pstr = ("bitwise" if par.get("bitwise") else f"{par.get('max_floored_rel_err', float('nan')):.1e}") if par else "—"
        if par and not par.get("pass"):
            pstr += " FAIL"
        rows.append(
            f"| {d['config']['workload']} | {d['dtype']} | {d.get('arithmetic', '')} | {fmt(d['value'])} | "
            f"{fmt(r.get('achieved'), '.0f')} | {fmt(r.get('frac'), '.3f')} | {fmt(r.get('frac_datasheet'), '.3f')} | "
            f"{d.get('flops_per_site', '—')} | {fmt(d.get('ai_flop_per_byte'), '.3f')} | {pstr} | "
            f"{fmt(r.get('kernel_avg_ms'), '.4f')} | {fmt(e2e.get('value'))} | "
            f"{fmt(cpu.get('value'))} ({cpu.get('kind', '—')}, {cpu.get('cores', '—')} core) | {fmt(ratio, '.3g')} |"
        )
    print("| workload | dtype | arithmetic | GPU site-ops/s | kernel GB/s (algorithmic) | of measured HBM | of datasheet 8000 GB/s "
          "| flop/site | flop/B | parity vs oracle | kernel ms | e2e site-ops/s | CPU baseline site-ops/s | GPU/CPU |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    print("\n".join(rows))


if __name__ == "__main__":
    main(sys.argv[1])
