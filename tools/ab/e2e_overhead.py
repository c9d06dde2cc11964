"""Host-side cost of one small drop-in call (4096 sites): where the e2e time of configs[0] goes."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1309_0551_b200 import _lib, kernels  # noqa: E402

dev = torch.device("cuda", 0)
n = 4096
res = {}
for dt in (torch.float32,):
    a_h = torch.randn((n, 3, 3, 2), dtype=dt).pin_memory()
    b_h = torch.randn((n, 3, 3, 2), dtype=dt).pin_memory()
    a_d, b_d, c_d = (torch.empty_like(a_h, device=dev) for _ in range(3))
    c_h = torch.empty_like(a_h).pin_memory()

    def loop(fn, reps=2000):
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps * 1e6

    res["copy_h2d_us"] = loop(lambda: a_d.copy_(a_h, non_blocking=True))
    res["copy_d2h_us"] = loop(lambda: c_h.copy_(c_d, non_blocking=True))
    res["smadd_wrapper_us"] = loop(lambda: kernels.scalar_mult_add_su3_matrix(a_d, b_d, 0.5, out=c_d))
    res["nn_wrapper_us"] = loop(lambda: kernels.mult_su3_nn(a_d, b_d, out=c_d))
    st = torch.cuda.current_stream().cuda_stream
    lib = _lib.load()
    pa, pb, pc = a_d.data_ptr(), b_d.data_ptr(), c_d.data_ptr()
    res["nn_raw_ctypes_us"] = loop(lambda: lib.su3g_mult_su3_nn_f32(pa, pb, pc, n, st))

    def step():
        a_d.copy_(a_h, non_blocking=True)
        b_d.copy_(b_h, non_blocking=True)
        kernels.mult_su3_nn(a_d, b_d, out=c_d)
        c_h.copy_(c_d, non_blocking=True)
    res["e2e_step_us"] = loop(step, 1000)
    a_np, b_np = a_h.numpy().copy(), b_h.numpy().copy()
    res["numpy_in_out_us"] = loop(lambda: kernels.mult_su3_nn(a_np, b_np), 300)
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
