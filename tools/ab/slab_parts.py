"""Time the pieces of one t-slab application on one GPU (64^3x16 f32): full sweep, interior slices
[1, nt-1), one boundary slice with halos, and the halo_w pack -- for the N > 1 weak-scaling budget."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(5)
for dt in (torch.float32, torch.float64):
    lat = Lattice4D(64, 64, 64, 16)
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, dt, dev, gen))
    v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, dt, dev, gen))
    out = v.empty_like()
    face = torch.zeros((6, lat.slice_sites), dtype=dt, device=dev)
    res = {"dtype": str(dt)}
    for variant, name in ((0, "auto"), (1, "generic")):
        _lib.set_option("nn_variant", variant)
        res[f"full_{name}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out))
        res[f"interior_{name}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(1, 15), v_hi=face, w_lo=face))
        res[f"boundary_lo_{name}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(0, 1), v_hi=face, w_lo=face))
        res[f"boundary_hi_{name}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(15, 16), v_hi=face, w_lo=face))
        res[f"kernel_{name}_boundary"] = _lib.last_kernel()
    _lib.set_option("nn_variant", 0)
    for r in (1, 4):
        _lib.set_option("sm_reserve", r)
        res[f"interior_auto_reserve{r}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(1, 15), v_hi=face, w_lo=face))
        res[f"interior_kernel_reserve{r}"] = _lib.last_kernel()
        res[f"full_auto_reserve{r}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out))
        res[f"full_kernel_reserve{r}"] = _lib.last_kernel()
    _lib.set_option("sm_reserve", 0)
    for c in (7, 14):
        _lib.set_option("nn_tma_chunk", c)
        res[f"interior_chunk{c}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(1, 15), v_hi=face, w_lo=face))
    _lib.set_option("nn_tma_chunk", 0)
    res["halo_w"] = timeit(lambda: sweeps.nn_halo_w(U, v, face))
    print(json.dumps(res))
