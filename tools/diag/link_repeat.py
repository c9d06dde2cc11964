"""Race check of the factored link walk: the same FMA-mode link product many times on the same links,
every output compared bit for bit with the first (a slot race shows as run-to-run differences, as the
ring-slot race of the NN walk did: profiles/r02/race_nn_ring_fma_nofence.log), both work-item schedules.

    python tools/diag/link_repeat.py [repetitions]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(11)
bad = 0
for dims in ((48, 48, 48, 48), (32, 32, 32, 24), (64, 64, 32, 16), (48, 12, 6, 7)):
    for dt in (torch.float64, torch.float32):
        lat = Lattice4D(*dims)
        U = Field.from_aos(lat, "mat4", inputs.random_links_torch(lat.volume, 4, dt, dev, gen))
        for chunk in (0, 5):
            _lib.set_option("link_chunk", chunk)
            first = None
            diffs = 0
            for r in range(reps):
                out = sweeps.link_product(U, 1.0 / 6.0, mode="fma").data.clone()
                torch.cuda.synchronize()
                if first is None:
                    first = out
                    kern = _lib.last_kernel()
                elif not torch.equal(first, out):
                    diffs += 1
            _lib.set_option("link_chunk", 0)
            print(f"{dims} {str(dt)[6:]} chunk {chunk}: {kern}: {diffs} of {reps - 1} repetitions differ", flush=True)
            bad += diffs
        del U
print("link_repeat:", "clean" if bad == 0 else f"{bad} DIFFERENCES")
sys.exit(1 if bad else 0)
