"""Launch each profiling target ONCE in one process, for a single ncu capture:

    ncu --set full -k regex:'k_link_rows|k_dslash|k_nn_tma' -c 3 ... python tools/prof_targets.py
Targets: link product 48^4 f64 exact (k_link_rows), even/odd dslash 64^3x16 f32 exact (k_dslash),
NN sweep 64^3x16 f32 exact (k_nn_tma, the headline kernel).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1309_0551_b200 import inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    lat = Lattice4D(48, 48, 48, 48)
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, torch.float64, dev, gen))
    sweeps.link_product(U, 1.0 / 6.0)
    del U
    lat = Lattice4D(64, 64, 64, 16)
    U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, torch.float32, dev, gen))
    v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, torch.float32, dev, gen))
    out = v.empty_like()
    sweeps.dslash(U, v, 0, out=out)
    sweeps.nn_sweep(U, v, out=out)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
