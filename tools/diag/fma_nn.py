"""Diagnose the 64^3x16 f32 FMA-mode NN sweep against the C oracle: which sites differ, repeatable or not."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import coracle  # noqa: E402
from oracle.compare import floored_rel_err  # noqa: E402
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402
from paper_1309_0551_b200.slab import CudaSlabKernels, SlabSweep  # noqa: E402

dims = tuple(int(a) for a in (sys.argv[1:5] or (64, 64, 64, 16)))
lat = Lattice4D(*dims)
dev = torch.device("cuda", 0)
for tdt in (torch.float32, torch.float64):
    gen = torch.Generator(device=dev)
    gen.manual_seed(1307)
    U_aos = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen)
    v_aos = inputs.random_vectors_torch(lat.volume, None, tdt, dev, gen)
    U, v = Field.from_aos(lat, "mat4", U_aos), Field.from_aos(lat, "vec", v_aos)
    U_h, v_h = U_aos.cpu().numpy(), v_aos.cpu().numpy()
    want = coracle.nn_sweep(U_h, v_h, dims)
    for variant in (0, 1, 3, 4):
        _lib.set_option("nn_variant", variant)
        for rep in range(3):
            try:
                out = sweeps.nn_sweep(U, v, mode="fma")
            except ValueError as e:
                print(tdt, variant, "n/a", e)
                break
            got = out.numpy()
            kern = _lib.last_kernel()
            err = floored_rel_err(got, want)
            ex = sweeps.nn_sweep(U, v, mode="exact").numpy()
            bitex = np.array_equal(ex, want)
            diff = np.abs(got.astype(np.float64) - want).reshape(lat.volume, -1).max(1)
            scale = np.abs(want).reshape(lat.volume, -1).max(1)
            bad = np.argwhere(diff > 1e-4 * np.maximum(scale, 1e-30)).ravel()
            print(f"{tdt} variant {variant} rep {rep} {kern}: err {err:.3g} exact-bitwise {bitex} bad sites {bad.size}",
                  flush=True)
            for b in bad[:6]:
                x = b % dims[0]; r = b // dims[0]; y = r % dims[1]; r //= dims[1]; z = r % dims[2]; t = r // dims[2]
                print("   site", b, (x, y, z, t), "got", got[b].ravel()[:4], "want", want[b].ravel()[:4])
        _lib.set_option("nn_variant", 0)
    slab = SlabSweep(U, kernels=CudaSlabKernels("fma"))
    o = v.empty_like()
    slab.apply(v, o)
    print(tdt, "slab fma err", floored_rel_err(o.numpy(), want), _lib.last_kernel(), flush=True)
