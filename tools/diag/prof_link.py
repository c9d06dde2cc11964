"""One 48^4 f64 link product per (variant, mode) given on the command line, for ncu: prof_link.py 3:fma 2:fma"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(5)
dt = torch.float32 if os.environ.get("DT") == "f32" else torch.float64
lat = Lattice4D(48, 48, 48, 48)
U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, dt, dev, gen))
for spec in sys.argv[1:]:
    v, m = spec.split(":")
    _lib.set_option("link_variant", int(v))
    sweeps.link_product(U, 1.0 / 6.0, mode=m)
    torch.cuda.synchronize()
    print(spec, _lib.last_kernel(), flush=True)
