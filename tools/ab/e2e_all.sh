cd "${GRAFT_REPO_ROOT:-.}"
for a in "" "--workload link --dtype f64" "--workload dslash --dtype f64" "--workload nn32" "--workload routine:scalar_mult_add_su3_matrix --sites 4096" "--workload routine:sub_four_su3_vecs --sites 65536" "--workload routine:mult_adj_su3_mat_4vec --sites 4096" "--workload dslash --layout soa"; do
  timeout 300 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('[$a]', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,4), d['e2e']['path'][:60])
except Exception: print('[$a] FAIL', l[-300:])" >> gpurun_out/e2e_all.txt
done
