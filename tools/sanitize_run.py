"""Every libsu3g kernel once, at small sizes, for compute-sanitizer (memcheck / synccheck / racecheck).

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

Covers the per-site stream kernels (all fifteen routines, both precisions), the layout transforms, the
seeded fill, the NN sweep kernels (ring walk, f32 TMA walk, generic, t-slab edges / halo pack), the
dslash (SoA parity kernels, checkerboarded fields), the link product (rows gather, row-split walk, factored pair walk), the
one-rank P2P boundary protocol and the one-rank NCCL slab driver.  Every result is compared with the
CPU oracle, so a kernel that misbehaves under the tool is visible in the exit code too.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle import coracle  # noqa: E402
from oracle import routines as R  # noqa: E402
from paper_1309_0551_b200 import _lib, inputs, kernels, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402


def check(ok, what):
    if not ok:
        print("MISMATCH:", what, flush=True)
        sys.exit(3)


def main():
    torch.cuda.set_device(0)
    rng = inputs.config_rng(77)
    n = 1000 + 13
    for dt in (np.float32, np.float64):
        U = inputs.random_links(rng, n, 4, dtype=dt)
        v = inputs.random_vectors(rng, n, 4, dtype=dt)
        h = rng.standard_normal((n, 2, 3, 2)).astype(dt)
        ops = {
            "mult_su3_mat_vec": (U[:, 0], v[:, 0]), "mult_adj_su3_mat_vec": (U[:, 0], v[:, 0]),
            "mult_su3_nn": (U[:, 0], U[:, 1]), "mult_su3_na": (U[:, 0], U[:, 1]), "mult_su3_an": (U[:, 0], U[:, 1]),
            "mult_adj_su3_mat_vec_4dir": (U, v[:, 0]), "mult_su3_mat_vec_sum_4dir": (U, v),
            "scalar_mult_add_su3_matrix": (U[:, 0], U[:, 1], dt(0.5)), "add_su3_vector": (v[:, 0], v[:, 1]),
            "mult_su3_mat_hwvec": (U[:, 0], h), "mult_adj_su3_mat_hwvec": (U[:, 0], h),
            "mult_adj_su3_mat_4vec": (U, v[:, 0]), "scalar_mult_add_su3_vector": (v[:, 0], v[:, 1], dt(0.5)),
            "su3_projector": (v[:, 0], v[:, 1]),
        }
        for r, o in ops.items():
            got = kernels.KERNELS[r](*o)
            want = R.ALL_ROUTINES[r](*o)
            if r == "mult_adj_su3_mat_4vec":
                got = np.stack(got, 1) if isinstance(got, (tuple, list)) else got
            check(np.array_equal(np.asarray(got), np.asarray(want)), f"{r} {dt}")
        a = v[:, 0].copy()
        kernels.sub_four_su3_vecs(a, v[:, 1], v[:, 2], v[:, 3], v[:, 0])
        check(np.array_equal(a, R.sub_four_su3_vecs(v[:, 0], v[:, 1], v[:, 2], v[:, 3], v[:, 0])), "sub_four")

    # sweeps on small lattices, every kernel family
    for dims in ((64, 4, 4, 6), (32, 4, 6, 5), (48, 2, 4, 3), (8, 4, 4, 4)):
        V = int(np.prod(dims))
        for dt in (np.float32, np.float64):
            U = inputs.random_links(rng, V, 4, dtype=dt)
            v = inputs.random_vectors(rng, V, None, dtype=dt)
            want = coracle.nn_sweep(U, v, dims)
            for variant in (0, 1, 3, 4):
                _lib.set_option("nn_variant", variant)
                try:
                    got = sweeps.nn_sweep_aos(U, v, dims)
                except ValueError:
                    continue
                finally:
                    _lib.set_option("nn_variant", 0)
                check(np.array_equal(got, want), f"nn {dims} {dt} variant {variant}")
            if dt == np.float32 and dims[0] >= 32:
                for cfg in (1, 2, 3):
                    _lib.set_option("nn_variant", 4)
                    _lib.set_option("nn_ring_cfg", cfg)
                    try:
                        check(np.array_equal(sweeps.nn_sweep_aos(U, v, dims), want), f"ring cfg {cfg} {dims}")
                    except ValueError:
                        pass
                    finally:
                        _lib.set_option("nn_ring_cfg", 0)
                        _lib.set_option("nn_variant", 0)
            wl = coracle.link_product(U, dims, 1 / 6)
            for lv in (1, 3, 5):
                _lib.set_option("link_variant", lv)
                try:
                    for mode in ("exact", "fma") if lv < 4 else ("fma",):
                        got = sweeps.link_product_aos(U, dims, 1 / 6, mode=mode)
                        check(mode == "fma" or np.array_equal(got, wl), f"link {dims} {dt} {lv}")
                except ValueError:
                    pass
                finally:
                    _lib.set_option("link_variant", 0)
            if all(d % 2 == 0 for d in dims):
                for parity in (0, 1):
                    sweeps.dslash_aos(U, v, dims, parity)
                    sweeps.dslash_aos(U, v, dims, parity, layout="eo")

    # t-slab pieces: halo pack, edges, P2P one-rank protocol, native NCCL driver
    lat = Lattice4D(16, 4, 4, 6)
    for tdt in (torch.float32, torch.float64):
        dt = np.float32 if tdt == torch.float32 else np.float64
        U_h = inputs.random_links(rng, lat.volume, 4, dtype=dt)
        v_h = inputs.random_vectors(rng, lat.volume, None, dtype=dt)
        want = coracle.nn_sweep(U_h, v_h, lat.dims)
        U, v = Field.from_aos(lat, "mat4", U_h), Field.from_aos(lat, "vec", v_h)
        w = torch.empty((6, lat.slice_sites), dtype=tdt, device="cuda")
        sweeps.nn_halo_w(U, v, w)
        out = v.empty_like()
        sweeps.nn_sweep(U, v, out=out, t_range=(1, lat.nt - 1), v_hi=v.face(0).contiguous(), w_lo=w)
        wn = torch.empty_like(w)
        sweeps.nn_edges(U, v, out, v_hi=v.face(0).contiguous(), w_lo=w, w_next=wn)
        check(np.array_equal(out.numpy(), want), f"slab pieces {tdt}")
        from paper_1309_0551_b200.p2p import P2PSlabSweep

        sw = P2PSlabSweep(U)
        o2 = sw.apply_n(Field(lat, "vec", tdt, data=v.data.clone()), 2)
        check(np.array_equal(o2.numpy(), coracle.nn_sweep_iterated(U_h, v_h, lat.dims, 2)), f"p2p {tdt}")
        sw.check()
        sw.close()
        from paper_1309_0551_b200.comm import NativeComm, native_slab_apply

        with NativeComm(1, 0, NativeComm.unique_id()) as c:
            o3 = native_slab_apply(c, U, Field(lat, "vec", tdt, data=v.data.clone()), 2)
            check(np.array_equal(o3.numpy(), coracle.nn_sweep_iterated(U_h, v_h, lat.dims, 2)), f"native {tdt}")

    # device-resident SiteBuffer fill
    from paper_1309_0551_b200.sitebuffer import DeviceSiteBuffer

    buf = DeviceSiteBuffer(Lattice4D(4, 4, 4, 4), {"a": "mat", "b": "vec"}, precision="double")
    buf.randomize(5)
    torch.cuda.synchronize()
    print("sanitize_run: all kernels ran and matched the oracle", flush=True)


if __name__ == "__main__":
    main()
