"""Interleaved A/B of the t-slab interior sweep (64^3x16 f32, slices [1, 15)) under sm_reserve 0 / 1 / 4,
plus the full periodic sweep, so clock drift over the run hits every arm equally."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(5)
lat = Lattice4D(64, 64, 64, 16)
U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, torch.float32, dev, gen))
v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, torch.float32, dev, gen))
out = v.empty_like()
face = torch.zeros((6, lat.slice_sites), dtype=torch.float32, device=dev)
rows = []
for rep in range(4):
    for r in (0, 1, 4):
        _lib.set_option("sm_reserve", r)
        ti = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(1, 15), v_hi=face, w_lo=face))
        ki = _lib.last_kernel()
        tf = timeit(lambda: sweeps.nn_sweep(U, v, out=out))
        rows.append({"rep": rep, "reserve": r, "interior_us": round(ti, 1), "full_us": round(tf, 1), "kernel": ki})
        torch.cuda.synchronize()
_lib.set_option("sm_reserve", 0)
for row in rows:
    print(json.dumps(row))
