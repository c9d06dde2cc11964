"""One t-slab application's boundary work on one GPU (64^3x16): two single-slice sweeps + halo pack
(separate launches) vs the fused edges launch (both slices + next w_last), interleaved."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1309_0551_b200 import inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def timeit(fn, reps=30):
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
for dt in (torch.float32, torch.float64):
    lat = Lattice4D(64, 64, 64, 16)
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, dt, dev, gen))
    v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, dt, dev, gen))
    out = v.empty_like()
    face = torch.zeros((6, lat.slice_sites), dtype=dt, device=dev)
    wn = torch.empty_like(face)

    def separate():
        sweeps.nn_halo_w(U, v, wn)
        sweeps.nn_sweep(U, v, out=out, t_range=(0, 1), v_hi=face, w_lo=face)
        sweeps.nn_sweep(U, v, out=out, t_range=(15, 16), v_hi=face, w_lo=face)

    def fused():
        sweeps.nn_edges(U, v, out, v_hi=face, w_lo=face, w_next=wn)

    rows = []
    for rep in range(3):
        rows.append({"dtype": str(dt), "rep": rep, "separate_us": round(timeit(separate), 1), "fused_us": round(timeit(fused), 1)})
    for r in rows:
        print(json.dumps(r))
