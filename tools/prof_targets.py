"""Launch each bench workload's dominant kernel ONCE in one process, for a single ncu --set full capture:

    ncu --set full -k regex:'k_nn_ring|k_link|k_dslash' -c 8 -o prof python tools/prof_targets.py

Targets, in launch order (the default dispatch of each bench workload):
  nn-weak f32 / f64  64^3x16 NN sweep (k_nn_ring)               -- the headline kernel
  link f64           48^4 link product, exact and FMA
  dslash f32 / f64   64^3x16 even/odd dslash on checkerboarded fields (k_dslash_ring)
The kernel names print to stdout, so the capture order can be matched to traffic.json keys.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    lat = Lattice4D(64, 64, 64, 16)
    for dt, key in ((torch.float32, "f32"), (torch.float64, "f64")):
        U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, dt, dev, gen))
        v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, dt, dev, gen))
        out = v.empty_like()
        sweeps.nn_sweep(U, v, out=out)
        torch.cuda.synchronize()
        print(f"nn-weak/{key}", _lib.last_kernel(), flush=True)
        del U, v, out
    lat = Lattice4D(48, 48, 48, 48)
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, torch.float64, dev, gen))
    for mode in ("exact", "fma"):
        sweeps.link_product(U, 1.0 / 6.0, mode=mode)
        torch.cuda.synchronize()
        print(f"link/f64/{mode}", _lib.last_kernel(), flush=True)
    del U
    lat = Lattice4D(64, 64, 64, 16)
    for dt, key in ((torch.float32, "f32"), (torch.float64, "f64")):
        U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, dt, dev, gen)).to_eo()
        v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, dt, dev, gen)).to_eo()
        out = v.empty_like()
        sweeps.dslash(U, v, 0, out=out)
        torch.cuda.synchronize()
        print(f"dslash/{key}", _lib.last_kernel(), flush=True)
        del U, v, out


if __name__ == "__main__":
    main()
