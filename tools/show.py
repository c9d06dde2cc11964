import json, re, sys
for line in open(sys.argv[1]):
    m = re.match(r'\[(.*?)\] (.*)', line)
    if not m:
        continue
    tag, rest = m.group(1), m.group(2)
    try:
        d = json.loads(rest)
    except Exception:
        print(tag, rest[:300]); continue
    r = d['roofline']
    print(f"{tag:50s} value={d['value']:.3e} GB/s={r['achieved']:.0f} frac={r['frac']:.3f} kern_ms={r['kernel_avg_ms']:.4f}")
