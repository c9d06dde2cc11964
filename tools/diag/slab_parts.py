"""Time the pieces of one t-slab application on one GPU (64^3x16 per rank): interior ring launch with SMs
reserved, the fused boundary launch, the halo pack, and the full native slab schedule (self communicator)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.comm import NativeComm, native_slab_sweep  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


for tdt in (torch.float32, torch.float64):
    lat = Lattice4D(64, 64, 64, 16)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, tdt, dev, g))
    v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, tdt, dev, g))
    out = v.empty_like()
    F = lat.slice_sites
    vhi = v.face(0).contiguous()
    wlo = torch.empty((6, F), dtype=tdt, device=dev)
    wn = torch.empty_like(wlo)
    res = {}
    res["periodic"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out))
    for r in (0, 4):
        _lib.set_option("sm_reserve", r)
        res[f"interior r{r}"] = timeit(lambda: sweeps.nn_sweep(U, v, out=out, t_range=(1, 15), v_hi=vhi, w_lo=wlo))
        k = _lib.last_kernel()
    _lib.set_option("sm_reserve", 0)
    res["edges"] = timeit(lambda: sweeps.nn_edges(U, v, out, v_hi=vhi, w_lo=wlo, w_next=wn))
    res["pack"] = timeit(lambda: sweeps.nn_halo_w(U, v, wlo))
    _lib.set_option("sm_reserve", 4)
    with NativeComm(1, 0, NativeComm.unique_id()) as c:
        res["native slab (self)"] = timeit(lambda: native_slab_sweep(c, U, v, out))
    _lib.set_option("sm_reserve", 0)
    print(tdt, k, {a: round(b, 1) for a, b in res.items()}, flush=True)
