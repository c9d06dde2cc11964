"""Host-side tests that need no GPU: the C ABI library, the registry, shapes, errors."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_1309_0551_b200 import _lib, lattice, types, validation

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "su3g.h")).read()
    return sorted(set(re.findall(r"SU3G_API[^;(]*?\b(su3g_\w+)\s*\(", text)))


def test_header_declares_the_full_abi():
    syms = header_symbols()
    for r in types.ROUTINE_NAMES:  # all fifteen Table-1 routines (the packed 4vec form is the 4dir entry)
        for sfx in ("f32", "f64"):
            assert f"su3g_{r}_{sfx}" in syms
    assert "su3g_nn_sweep_f32" in syms and "su3g_link_product_f64" in syms
    assert len(syms) == len(_lib.SIGNATURES)
    assert set(syms) == set(_lib.SIGNATURES)


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name
    assert lib.su3g_abi_version() == 1


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_invalid_arguments_rejected_without_touching_the_device():
    lib = _lib.load()
    # negative site count, null pointers -> SU3G_EINVAL before any CUDA call
    assert lib.su3g_mult_su3_mat_vec_f32(None, None, None, -1, None) == _lib.SU3G_EINVAL
    assert b"negative" in lib.su3g_last_error()
    assert lib.su3g_nn_sweep_f32(None, None, None, 0, 4, 4, 4, 0, 4, None, None, 0, None) == _lib.SU3G_EINVAL
    assert lib.su3g_nn_sweep_f32(None, None, None, 4, 4, 4, 4, 0, 4, None, None, 9, None) == _lib.SU3G_EINVAL
    assert lib.su3g_link_product_f64(None, None, 4, 4, 4, 4, 0.5, 7, None) == _lib.SU3G_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.SU3G_EINVAL, "x")
    assert lib.su3g_sub_four_su3_vecs_f32(None, None, None, None, None, -2, None) == _lib.SU3G_EINVAL
    assert lib.su3g_mult_adj_su3_mat_4vec_f64(None, None, None, None, None, None, -1, None) == _lib.SU3G_EINVAL
    # checkerboarded layout / dslash: odd extents, bad parity, null pointers
    assert lib.su3g_soa_to_eo_f32(None, None, 4, 4, 4, 3, 6, None) == _lib.SU3G_EINVAL
    assert b"even" in lib.su3g_last_error()
    assert lib.su3g_eo_to_soa_f64(None, None, 4, 4, 4, 4, 6, None) == _lib.SU3G_EINVAL
    assert lib.su3g_dslash_eo_f32(None, None, None, 4, 4, 4, 4, 2, 0, None) == _lib.SU3G_EINVAL
    assert lib.su3g_dslash_eo_f64(None, None, None, 4, 4, 4, 4, 0, 0, None) == _lib.SU3G_EINVAL
    # zero sites is a valid no-op
    assert lib.su3g_mult_su3_nn_f64(None, None, None, 0, None) == _lib.SU3G_OK
    assert lib.su3g_sub_four_su3_vecs_f64(None, None, None, None, None, 0, None) == _lib.SU3G_OK


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_tuning_knobs_validate_names_and_ranges_without_a_device():
    """su3g_set_option (include/su3g.h): every documented knob accepts its range, rejects the rest
    (the removed ring link walk included), and restores its default."""
    lib = _lib.load()
    ok = {"nn_variant": (0, 1, 3, 4), "link_variant": (0, 1, 3, 5), "dslash_eo_variant": (0, 1, 2),
          "dslash_eo_ring_cfg": (0, 1, 2), "nn_ring_cfg": (0, 1, 2, 3, 4),
          "sm_reserve": (0, 4), "link_chunk": (0, 12, 4096), "nn_ring_columns": (0, 1)}
    bad = {"nn_variant": (2, 5), "link_variant": (2, 4, 6, -1), "dslash_eo_variant": (3, -1),
           "dslash_eo_ring_cfg": (3,), "nn_ring_cfg": (5,), "sm_reserve": (-1, 65),
           "link_chunk": (-1, 4097), "nn_ring_columns": (-1, 2), "link_pair_prefetch": (0,), "link_zdown": (0,)}
    try:
        for name, vals in ok.items():
            for v in vals:
                assert lib.su3g_set_option(name.encode(), v) == _lib.SU3G_OK, (name, v)
        for name, vals in bad.items():
            for v in vals:
                assert lib.su3g_set_option(name.encode(), v) == _lib.SU3G_EINVAL, (name, v)
        lib.su3g_set_option(b"link_variant", 2)
        assert b"removed" in lib.su3g_last_error()
        assert lib.su3g_set_option(b"no_such_knob", 0) == _lib.SU3G_EINVAL
    finally:
        for name, default in (("nn_variant", 0), ("link_variant", 0), ("dslash_eo_variant", 0),
                              ("dslash_eo_ring_cfg", 0), ("nn_ring_cfg", 0),
                              ("sm_reserve", 0), ("link_chunk", 0), ("nn_ring_columns", 1)):
            lib.su3g_set_option(name.encode(), default)


def test_no_cpu_fallback():
    from paper_1309_0551_b200 import kernels

    a = np.zeros((2, 3, 3, 2), np.float32)
    b = np.zeros((2, 3, 2), np.float32)
    with pytest.raises(RuntimeError, match="CUDA device"):
        kernels.mult_su3_mat_vec(a, b)


def test_shape_errors_match_reference_conventions():
    from paper_1309_0551_b200 import kernels

    a = np.zeros((4, 3, 3, 2), np.float32)
    b = np.zeros((4, 3, 2), np.float32)
    with pytest.raises(ValueError):
        kernels.mult_su3_mat_vec(b, b)  # wrong per-object shape
    with pytest.raises(ValueError):
        kernels.mult_su3_nn(a, b)
    with pytest.raises(ValueError):
        kernels.mult_su3_mat_vec(a, b[:3])  # batch shapes disagree
    with pytest.raises(ValueError):
        kernels.mult_su3_mat_vec(a, b.astype(np.float64))  # mixed precision (deliberate tightening)
    with pytest.raises(ValueError):
        kernels.mult_su3_mat_vec(a, b, out=np.zeros((4, 3, 3, 2), np.float32))
    with pytest.raises(ValueError):
        kernels.apply("mult_su3_zz", a, b)
    with pytest.raises(ValueError):
        kernels.batch_apply("mult_su3_nn", [a, a[:3]])
    with pytest.raises(ValueError):
        kernels.batch_apply("mult_su3_nn", [a, a], count=9)


def test_alias_check_under_debug_validation():
    from paper_1309_0551_b200 import kernels

    a = np.zeros((4, 3, 3, 2), np.float32)
    b = np.zeros((4, 3, 2), np.float32)
    validation.debug_validation(True)
    try:
        with pytest.raises(ValueError, match="aliases"):
            kernels.mult_su3_mat_vec(a, b, out=b)
        t = torch.zeros(10)
        with pytest.raises(ValueError, match="aliases"):
            validation.check_no_alias(t[2:6], t[4:8])
        validation.check_no_alias(t[0:4], t[4:8])
    finally:
        validation.debug_validation(False)


def test_registry_and_batch_count():
    assert set(types.HOT_ROUTINE_NAMES) == set(_lib.HOT_ROUTINES) | {"scalar_mult_add_su3_matrix"}
    assert len(types.ROUTINE_NAMES) == 15 and set(types.HOT_ROUTINE_NAMES) <= set(types.ROUTINE_NAMES)
    assert types.routine_spec("sub_four_su3_vecs").in_place
    spec = types.routine_spec("scalar_mult_add_su3_matrix")
    a = np.zeros((5, 3, 3, 2))
    assert types.batch_count(spec, [a, a, 0.5]) == 5
    assert types.batch_count(spec, [a, a, np.zeros(5)]) == 5
    assert types.batch_count(types.routine_spec("mult_su3_nn"), [a[:0], a[:0]]) == 0
    with pytest.raises(ValueError):
        types.routine_spec("nope")
    assert types.dtype_for("single") == np.float32
    with pytest.raises(ValueError):
        types.dtype_for(np.int32)


def test_lattice_matches_reference_numbering():
    lat = lattice.Lattice4D(4, 4, 4, 4)
    assert lat.site_index((1, 0, 0, 0)) == 1
    assert lat.site_index((0, 1, 0, 0)) == 4
    assert lat.site_index((0, 0, 1, 0)) == 16
    assert lat.site_index((0, 0, 0, 1)) == 64
    assert lat.neighbor(lat.site_index((3, 0, 0, 0)), "+x") == 0
    assert lat.neighbor(0, "-t") == lat.site_index((0, 0, 0, 3))
    lat2 = lattice.Lattice4D(2, 3, 4, 5)
    for s in range(lat2.volume):
        assert lat2.site_index(lat2.site_coord(s)) == s
        for d in lattice.DIRECTIONS:
            opp = ("-" if d[0] == "+" else "+") + d[1]
            assert lat2.neighbor(lat2.neighbor(s, d), opp) == s
    assert lattice.Lattice4D(8, 8, 8, 16).slab(4, 1).dims == (8, 8, 8, 4)
    with pytest.raises(ValueError):
        lattice.Lattice4D(8, 8, 8, 6).slab(4, 0)
    with pytest.raises(ValueError):
        lattice.Lattice4D(0, 1, 1, 1)


def test_lattice_numbering_agrees_with_oracle_shift():
    from oracle import sweeps as S

    dims = (3, 4, 5, 6)
    lat = lattice.Lattice4D(*dims)
    idx = np.arange(lat.volume).reshape(-1, 1)
    for mu, axis in enumerate("xyzt"):
        up = S.shift(idx, dims, mu, +1)[:, 0]
        assert all(up[s] == lat.neighbor(s, "+" + axis) for s in range(0, lat.volume, 7))


def test_input_generators_are_special_unitary():
    from paper_1309_0551_b200 import inputs

    U = inputs.random_links(inputs.config_rng(1), 300, 4)
    u = U[..., 0] + 1j * U[..., 1]
    eye = np.einsum("...ij,...kj->...ik", u, u.conj())
    assert np.abs(eye - np.eye(3)).max() < 1e-13
    assert np.abs(np.linalg.det(u) - 1).max() < 1e-13
    # deterministic per seed
    a = inputs.random_vectors(np.random.default_rng(5), 10, None)
    b = inputs.random_vectors(np.random.default_rng(5), 10, None)
    assert np.array_equal(a, b)


def test_register_with_su3bench_plugin_registry():
    """The b200 record slots into the reference's own registry (backends.py:19-31), harness config accepts it."""
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference package not present (GPU box)")
    import sys

    sys.path.insert(0, ref)
    try:
        import su3bench.backends as rb
        from su3bench.bench import BenchConfig

        from paper_1309_0551_b200 import backends, kernels

        rec = backends.register_with_su3bench()
        try:
            assert rb.get_backend("b200") is rec
            assert isinstance(rec, rb.Backend)
            assert set(rec.kernels) == set(kernels.KERNELS)
            BenchConfig(routine="mult_su3_nn", backend="b200")  # validated through get_backend (bench.py:66)
        finally:
            rb._BACKENDS.pop("b200", None)
            rb.BACKEND_NAMES = tuple(rb._BACKENDS)
    finally:
        sys.path.remove(ref)


def test_bench_reference_arm_contract(capsys):
    """bench.py --impl reference prints one JSON line with the contract keys (runs on CPU)."""
    import json

    import bench

    bench.main(["--impl", "reference", "--steps", "1", "--warmup", "3", "--dims", "16,16,16,4"])
    line = capsys.readouterr().out.strip().splitlines()[-1]
    d = json.loads(line)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config5-weak")


def test_bench_rejects_short_warmup():
    import bench

    with pytest.raises(SystemExit):
        bench.parse_args(["--warmup", "2"])


def _pcg_model(state, inc, skip, n):
    """Pure-Python PCG64 XSL-RR + uniform(-1, 1), with the jump-ahead fill.cu uses."""
    M128, MULT = (1 << 128) - 1, 0x2360ED051FC65DA44385DF649FCCF645

    def jump(delta):
        am, ap, cm, cp = 1, 0, MULT, inc
        while delta:
            if delta & 1:
                am, ap = (am * cm) & M128, (ap * cm + cp) & M128
            cp, cm = ((cm + 1) * cp) & M128, (cm * cm) & M128
            delta >>= 1
        return am, ap

    a, c = jump(skip + 1)
    s = (a * state + c) & M128
    out = []
    for _ in range(n):
        x = ((s >> 64) ^ s) & ((1 << 64) - 1)
        r = s >> 122
        x = ((x >> r) | (x << (64 - r))) & ((1 << 64) - 1) if r else x
        out.append(-1.0 + 2.0 * ((x >> 11) * (1.0 / 9007199254740992.0)))
        s = (s * MULT + inc) & M128
    return np.array(out)


@pytest.mark.parametrize("skip", [0, 1, 7, 1000, 123456789])
def test_pcg64_jump_ahead_model_matches_numpy(skip):
    """The jump-ahead + output function of csrc/fill.cu, modelled in Python, reproduces numpy's stream."""
    from paper_1309_0551_b200.sitebuffer import pcg64_seed_state

    state, inc = pcg64_seed_state(2024)
    rng = np.random.default_rng(2024)
    rng.bit_generator.advance(skip)
    assert np.array_equal(_pcg_model(state, inc, skip, 5), rng.uniform(-1.0, 1.0, size=5))


def test_device_sitebuffer_rejects_bad_alignment():
    from paper_1309_0551_b200.sitebuffer import DeviceSiteBuffer

    with pytest.raises(ValueError, match="power of two"):
        DeviceSiteBuffer(lattice.Lattice4D(2, 2, 2, 2), {"a": "vec"}, alignment=12)


def test_comm_abi_without_a_gpu():
    """Unique ids come from NCCL without a device; bad arguments are rejected before any CUDA call."""
    from paper_1309_0551_b200.comm import NativeComm

    lib = _lib.load()
    uid = NativeComm.unique_id()
    assert len(uid) == _lib.SU3G_COMM_ID_BYTES and any(uid)
    h = ctypes.c_void_p()
    assert lib.su3g_comm_init(2, 2, uid, ctypes.byref(h)) == _lib.SU3G_EINVAL
    assert lib.su3g_comm_init(1, 0, None, ctypes.byref(h)) == _lib.SU3G_EINVAL
    assert lib.su3g_comm_destroy(None) == _lib.SU3G_OK
    assert lib.su3g_comm_check(None, 1000) == _lib.SU3G_EINVAL
    with pytest.raises(RuntimeError):  # NCCL failures surface as RuntimeError, argument errors as ValueError
        _lib.check(_lib.SU3G_ENCCL, "x")
    assert lib.su3g_slab_nn_sweep_f32(None, None, None, None, 4, 4, 4, 4, 0, None) == _lib.SU3G_EINVAL
    with pytest.raises(ValueError, match="128"):
        NativeComm(1, 0, b"short")


def test_p2p_abi_argument_checks():
    lib = _lib.load()
    nb = lib.su3g_p2p_window_bytes(64, 64, 64, 4)
    assert nb == 4 * 6 * 64**3 * 4 + 128 and lib.su3g_p2p_ctrl_offset(64, 64, 64, 4) == nb - 128
    assert lib.su3g_p2p_window_bytes(0, 4, 4, 4) == -1 and lib.su3g_p2p_window_bytes(4, 4, 4, 2) == -1
    assert lib.su3g_p2p_nn_sweep_f32(None, None, None, 4, 4, 4, 4, None, None, None, 0, 0, None) == _lib.SU3G_EINVAL
    assert lib.su3g_p2p_prime_f64(None, None, 4, 4, 4, 4, None, None, None, 0, 0, None) == _lib.SU3G_EINVAL
    assert lib.su3g_ipc_get_handle(None, None) == _lib.SU3G_EINVAL
    assert lib.su3g_ipc_close(None) == _lib.SU3G_OK


def _build_c_demo(tmp_path):
    """Compile tests/c/abi_demo.c as plain C11 against include/su3g.h and libsu3g.so."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = tmp_path / "abi_demo"
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = [cc, "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "c", "abi_demo.c"), "-o", str(exe), "-L", libdir, "-lsu3g",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_host_program_against_the_abi(tmp_path):
    """A C program (no Python, no torch) includes su3g.h, links libsu3g.so and exercises the ABI."""
    import subprocess

    exe = _build_c_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert "abi_demo: ok" in r.stdout


def test_field_layout_validation_without_a_gpu():
    """The checkerboarded ('eo') layout needs even extents; unknown layouts are rejected (before any allocation)."""
    from paper_1309_0551_b200.lattice import Field, Lattice4D

    with pytest.raises(ValueError, match="even"):
        Field(Lattice4D(4, 4, 4, 3), "vec", layout="eo")
    with pytest.raises(ValueError, match="layout"):
        Field(Lattice4D(4, 4, 4, 4), "vec", layout="aos")


@pytest.mark.parametrize("columns", [0, 1])
def test_walk_schedule_covers_every_block_slice_exactly_once(columns):
    """The persistent t-walks' work-item schedule (csrc/sweep_common.cuh pick_schedule / schedule_item,
    through su3g_walk_schedule): for both the uniform and the columns form, the items partition
    blocks x slices exactly, whole-column items come first, and the columns form never takes more
    rounds of CTAs (weighted by item length + prologue) than the uniform one it replaces."""
    lib = _lib.load()
    rng = np.random.default_rng(1309)
    cases = [(768, 48, 148), (1024, 16, 296), (1024, 16, 148), (1024, 14, 296), (256, 32, 592), (320, 3, 148),
             (1, 1, 148), (148, 7, 148), (149, 5, 148)]
    cases += [(int(rng.integers(1, 1500)), int(rng.integers(1, 130)), int(rng.choice([148, 296, 444, 592])))
              for _ in range(40)]
    blk, n_full = ctypes.c_int64(), ctypes.c_int64()
    t0, t1, chunk = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()

    def cost(nblocks, L, G, cols, prologue):
        n = lib.su3g_walk_schedule(nblocks, L, G, int(prologue * 10), cols, -1, None, None, None,
                                   ctypes.byref(n_full), ctypes.byref(chunk))
        rounds_full = n_full.value // G
        rest = n - n_full.value
        return rounds_full * (L + prologue) + -(-rest // G) * (chunk.value + prologue) if rest else rounds_full * (L + prologue)

    for nblocks, L, G in cases:
        n = lib.su3g_walk_schedule(nblocks, L, G, 5, columns, -1, None, None, None, ctypes.byref(n_full),
                                   ctypes.byref(chunk))
        assert n > 0 and 1 <= chunk.value <= L and 0 <= n_full.value <= nblocks, (nblocks, L, G)
        assert n_full.value % G == 0 and (columns or n_full.value == 0)
        seen = np.zeros((nblocks, L), dtype=np.int32)
        for item in range(n):
            assert lib.su3g_walk_schedule(nblocks, L, G, 5, columns, item, ctypes.byref(blk), ctypes.byref(t0),
                                          ctypes.byref(t1), None, None) == n
            assert 0 <= blk.value < nblocks and 0 <= t0.value < t1.value <= L, (nblocks, L, G, item)
            if item < n_full.value:
                assert (blk.value, t0.value, t1.value) == (item, 0, L)
            seen[blk.value, t0.value:t1.value] += 1
        assert (seen == 1).all(), (nblocks, L, G, columns)
        if columns:
            assert cost(nblocks, L, G, 1, 0.5) <= cost(nblocks, L, G, 0, 0.5) + 1e-9, (nblocks, L, G)
    assert lib.su3g_walk_schedule(0, 4, 148, 5, 1, -1, None, None, None, None, None) == -1
