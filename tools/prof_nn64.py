"""One process, NN sweep 64^3x16 f64 exact: generic kernel then the TMA64 variant (for one ncu capture),
and the dslash f32 (k_dslash).  Usage: ncu ... -k regex:'k_nn_sweep|k_nn_tma64|k_dslash' python tools/prof_nn64.py"""
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
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, torch.float64, dev, gen))
    v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, torch.float64, dev, gen))
    out = v.empty_like()
    for variant in (1, 5):
        _lib.set_option("nn_variant", variant)
        for _ in range(2):
            sweeps.nn_sweep(U, v, out=out)
    _lib.set_option("nn_variant", 0)
    del U, v, out
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, torch.float32, dev, gen))
    v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, torch.float32, dev, gen))
    out = v.empty_like()
    for _ in range(2):
        sweeps.dslash(U, v, 0, out=out)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
