"""Benchmark driver for the B200 SU(3) hot path (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload nn-weak|nn-strong|nn32|link|routine:<name>] [--dtype f32|f64]

Default workload = BASELINE configs[4], weak-scaling variant: the periodic
nearest-neighbour sweep on a 64^3 x 16*N lattice, t sharded into one 64^3x16
slab per GPU (one-site halos over NCCL), complex64; one step = 10 repeated
applications v <- D v on device-resident fields.  `value` is whole-job
site-ops/s (sites x applications / s, max over ranks); `e2e` is the same
metric through the reference-facing path with host (AoS, pinned) buffers
and the H2D/D2H copies inside the timed region; `roofline` is the NN-sweep
kernel's algorithmic HBM bytes / CUDA-event duration against the measured
copy bandwidth in MEASURED_PEAKS.json.

--impl reference times the reference's own algorithm on the host CPU (the
pinned numpy restatement in oracle/, parallelised over t-slabs with all host
threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SU(3) site-ops/s and HBM GB/s as % of peak (fp32/fp64), 1–8 GPUs"
UNIT = "site-ops/s"
FALLBACK_HBM_GBS = 6650.0
DATASHEET_HBM_GBS = 8000.0  # B200 datasheet HBM3e bandwidth (reported beside the measured peak)

# algorithmic (compulsory) HBM bytes per site: read each input object once, write each output once
NN_BYTES = {"f32": 336, "f64": 672}        # U 72 reals + v 6 + out 6
LINK_BYTES = {"f32": 360, "f64": 720}      # U 72 + acc 18
# even/odd dslash, per lattice site per one-parity launch: all of U (forward links of the
# output sites + backward links of their neighbours) + v on the other half + out on this half
DSLASH_BYTES = {"f32": 288 + 24, "f64": 576 + 48}
def _routine_layout():
    """routine -> (reals per site of each array operand, reals per site of the result), from the registry."""
    from paper_1309_0551_b200 import types as T

    out = {}
    for name, spec in T.ROUTINES.items():
        out[name] = ([T.REALS[k] for k in spec.operands if k != "scalar"], T.REALS[spec.result])
    return out


ROUTINE_LAYOUT = _routine_layout()
# (in reals, out reals) per site -- algorithmic bytes = (in + out) x element size
ROUTINE_REALS = {r: (sum(ins), res) for r, (ins, res) in ROUTINE_LAYOUT.items()}
SMADD_ROUTINES = ("scalar_mult_add_su3_matrix", "scalar_mult_add_su3_vector")


def parse_args(argv=None):
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--workload", default="nn-weak")
    p.add_argument("--dtype", choices=["f32", "f64"], default=None)
    p.add_argument("--applications", type=int, default=10)
    p.add_argument("--mode", choices=["exact", "fma"], default=None,
                   help="SU(3) product arithmetic: exact = reference association, bit-identical (default "
                        "for the NN sweep); fma = FMA chains within the north-star tolerance")
    p.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e measurement")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-parity", action="store_true", help="skip the parity check of the timed path against the C oracle")
    p.add_argument("--no-slab-probe", action="store_true",
                   help="skip the one-GPU run of the N>1 per-rank t-slab schedule (nn workloads, N=1)")
    p.add_argument("--sites", type=int, default=64**4, help="sites for routine:<name> workloads")
    p.add_argument("--streams", type=int, default=16,
                   help="routine:<name> workloads below 2^20 sites: concurrent graph branches the independent "
                        "batch calls are spread over (1 = one serial chain; 16 measured best at 4096 sites)")
    p.add_argument("--halo", choices=["nccl", "p2p"], default="nccl",
                   help="t-slab halo transport of the nn-* workloads: NCCL send/recv overlapped with the interior "
                        "(default), or the fused boundary kernel pushing halos over NVLink (csrc/p2p.cu)")
    p.add_argument("--layout", choices=("eo", "soa"), default="eo",
                   help="dslash workload: checkerboarded (eo) fields and su3g_dslash_eo, or t-sliced SoA fields")
    p.add_argument("--dims", default=None,
                   help="experiments only: override the lattice nx,ny,nz,nt of nn-*/dslash/link workloads "
                        "(for nn-weak, nt is per GPU)")
    args = p.parse_args(argv)
    if args.warmup < 3:
        p.error("--warmup must be >= 3")
    if args.dtype is None:
        args.dtype = "f64" if args.workload == "link" else "f32"
    if args.mode is None:
        args.mode = os.environ.get("SU3G_LINK_MODE", "exact") if args.workload == "link" else "exact"
    return args


# ----------------------------------------------------------------------------
# workload geometry
# ----------------------------------------------------------------------------

def workload_config(args, world):
    cfg = _workload_config(args, world)
    if args.dims and cfg["kind"] in ("nn", "dslash", "link"):
        d = tuple(int(x) for x in args.dims.split(","))
        if len(d) != 4:
            raise SystemExit("--dims needs nx,ny,nz,nt")
        cfg["global_dims"] = d[:3] + (d[3] * (world if args.workload == "nn-weak" else 1),)
        cfg["name"] += f" [dims override {d}]"
    return cfg


def _workload_config(args, world):
    w = args.workload
    if w == "nn-weak":
        return dict(kind="nn", global_dims=(64, 64, 64, 16 * world), apps=args.applications,
                    name=f"config5-weak: periodic NN sweep 64^3x16*N t-slabs, {args.applications} applications/step")
    if w == "nn-strong":
        return dict(kind="nn", global_dims=(64, 64, 64, 128), apps=args.applications,
                    name=f"config5-strong: periodic NN sweep 64^3x128 t-slabs, {args.applications} applications/step")
    if w == "nn32":
        return dict(kind="nn", global_dims=(32, 32, 32, 32), apps=1, name="config2: periodic NN sweep 32^4, 1 application/step")
    if w == "link":
        return dict(kind="link", global_dims=(48, 48, 48, 48), apps=1, name="config3: link-product sweep 48^4, 1 sweep/step")
    if w == "dslash":
        return dict(kind="dslash", global_dims=(64, 64, 64, 16), apps=1,
                    name="8(f) f3: even/odd dslash 64^3x16, D_eo + D_oe (both parities) per step")
    if w.startswith("routine:"):
        r = w.split(":", 1)[1]
        if r not in ROUTINE_REALS:
            raise SystemExit(f"unknown routine {r!r}")
        return dict(kind="routine", routine=r, nsites=args.sites, apps=1,
                    name=f"{r} streaming batch of {args.sites} sites (roofline run for configs[0]/[1])")
    raise SystemExit(f"unknown workload {w!r}")


# ----------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ----------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.ok = False
        self.period = period_s
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:  # noqa: BLE001
            pass

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self.ok and self._t is not None:
            self._sample()
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        names = [n for n, bit in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _compute_floor(cfg, args, bytes_per_launch, kern_avg_ms, kernel=""):
    """Exact-mode FP-pipe time of one launch (every flop one FMUL/FADD or DMUL/DADD, flops.py) beside the
    HBM time of its algorithmic bytes: which roof binds.  FMA mode: only the link product (its factored
    form's 990 fused instructions per site); None for the other FMA-mode sweeps and the routines."""
    from paper_1309_0551_b200 import flops as _flops

    if cfg["kind"] == "link" and args.mode == "fma" and kern_avg_ms and (kernel or "").startswith("k_link_fact"):
        # the factored walk issues 990 fused FP instructions per site (flops.LINK_FACTORED_FP_INSTRUCTIONS)
        sites = bytes_per_launch / _flops.intensity("link", args.dtype)["bytes_per_site"]
        fp_ms = _flops.fma_floor_s(_flops.LINK_FACTORED_FP_INSTRUCTIONS, args.dtype, int(sites)) * 1e3
        hbm_ms = bytes_per_launch / (peak_hbm()[0] * 1e9) * 1e3
        return {"fp_pipe_ms": fp_ms, "hbm_ms": hbm_ms, "bound": "fp-pipe" if fp_ms > hbm_ms else "hbm",
                "max_hbm_frac": min(1.0, hbm_ms / fp_ms), "frac_of_binding_roof": max(fp_ms, hbm_ms) / kern_avg_ms,
                "fp_instructions_per_site": _flops.LINK_FACTORED_FP_INSTRUCTIONS,
                "pipe": "FP32 128 / FP64 64 lanes per SM per clock x 148 SMs x 1.965 GHz, factored form: "
                        "nine 3x3 complex products of 108 FMAs + 18 multiplies per site"}
    if cfg["kind"] not in ("nn", "link", "dslash") or args.mode != "exact" or not kern_avg_ms:
        return None
    per_site = _flops.intensity(cfg["kind"], args.dtype)["bytes_per_site"]
    if cfg["kind"] == "dslash":
        per_site = DSLASH_BYTES[args.dtype]
    sites = bytes_per_launch / per_site
    if cfg["kind"] == "dslash":
        sites /= 2  # one parity launch computes half of the sites
    fp_ms = _flops.compute_floor_s(cfg["kind"], args.dtype, int(sites)) * 1e3
    hbm_ms = bytes_per_launch / (peak_hbm()[0] * 1e9) * 1e3
    return {"fp_pipe_ms": fp_ms, "hbm_ms": hbm_ms, "bound": "fp-pipe" if fp_ms > hbm_ms else "hbm",
            "max_hbm_frac": min(1.0, hbm_ms / fp_ms), "frac_of_binding_roof": max(fp_ms, hbm_ms) / kern_avg_ms,
            "pipe": "FP32 128 / FP64 64 lanes per SM per clock x 148 SMs x 1.965 GHz, one instruction per flop"}


def traffic_for(workload: str, dtype: str, mode: str, kernel: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from a committed ncu --set full
    capture (profiles/traffic.json), or None when no capture of THIS kernel exists: an entry counts
    only if the kernel that ran starts with the kernel the capture measured."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            table = json.load(f)
    except Exception:  # noqa: BLE001
        return None
    for key in (f"{workload}/{dtype}/{mode}", f"{workload}/{dtype}"):
        e = table.get(key)
        if isinstance(e, dict) and kernel and kernel.startswith(e.get("kernel", "\0")):
            return e.get("bytes")
    return None


# ----------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------

def init_dist(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "b200" or world > 1:
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        if args.impl == "b200":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return rank, world, local


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world, device=None):
    if world > 1:
        import torch.distributed as dist

        if device is not None:
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


# ----------------------------------------------------------------------------
# the B200 arm
# ----------------------------------------------------------------------------

def run_b200(args, rank, world, local):
    import torch

    from paper_1309_0551_b200 import inputs, kernels, sweeps
    from paper_1309_0551_b200.lattice import Field, Lattice4D
    from paper_1309_0551_b200.slab import CudaSlabKernels, SlabSweep

    cfg = workload_config(args, world)
    dev = torch.device("cuda", local)
    # A/B tuning knobs (su3g_set_option), from the environment
    from paper_1309_0551_b200 import _lib as _l

    for env, opt in (("SU3G_NN_VARIANT", "nn_variant"), ("SU3G_CHUNK_PROLOGUE_X10", "chunk_prologue_x10"),
                     ("SU3G_NN_TMA_THREADS", "nn_tma_threads"), ("SU3G_SWEEP_ZC", "sweep_zc"),
                     ("SU3G_SWEEP_L2_HINTS", "sweep_l2_hints"), ("SU3G_NN_TMA_L2_HINTS", "nn_tma_l2_hints"),
                     ("SU3G_NN_TMA_CHUNK", "nn_tma_chunk"), ("SU3G_DSLASH_EO_ZC", "dslash_eo_zc"),
                     ("SU3G_DSLASH_EO_HINTS", "dslash_eo_hints"), ("SU3G_NN_RING_CFG", "nn_ring_cfg"),
                     ("SU3G_LINK_VARIANT", "link_variant"),
                     ("SU3G_LINK_CHUNK", "link_chunk"), ("SU3G_NN_RING_COLUMNS", "nn_ring_columns"),
                     ("SU3G_DSLASH_EO_VARIANT", "dslash_eo_variant"), ("SU3G_DSLASH_EO_RING_CFG", "dslash_eo_ring_cfg")):
        if os.environ.get(env):
            _l.set_option(opt, int(os.environ[env]))
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    gen = torch.Generator(device=dev)
    gen.manual_seed(inputs.SEED + 7919 * rank)
    stream = torch.cuda.current_stream(dev)
    launches_per_step = 0
    launches_per_event = 1
    dominant_events = []  # (start, end) pairs around the dominant kernel

    if cfg["kind"] == "nn":
        gd = cfg["global_dims"]
        glat = Lattice4D(*gd)
        lat = glat.slab(world, rank)
        U_aos = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen)
        v_aos = inputs.random_vectors_torch(lat.volume, None, tdt, dev, gen)
        U = Field.from_aos(lat, "mat4", U_aos)
        v0 = Field.from_aos(lat, "vec", v_aos)
        va, vb = v0.empty_like(), v0.empty_like()
        ntl = lat.nt
        apps = cfg["apps"]
        # one step = `apps` chained applications v <- D v starting from the step's input field v0 (never
        # overwritten): the first reads v0, the rest ping-pong between va and vb.  Starting every step
        # from v0 keeps the values finite (|D| ~ 10: 10 applications, not thousands, compound).
        last = [v0]
        if args.halo == "p2p":
            from paper_1309_0551_b200.p2p import P2PSlabSweep

            p2p = P2PSlabSweep(U, mode=args.mode)
            per_launch_sites = lat.volume  # timed unit: one application (boundary + interior launches)
            launches_per_app = 2 if ntl > 2 else 1
            extra_launches = 1  # the first application of a step primes the halos of the fresh source

            def run_step(record=False):
                src = v0
                for i in range(apps):
                    dst = va if i % 2 == 0 else vb
                    if record:
                        with _EventTimer(stream, dominant_events):
                            p2p.apply(src, dst, chain=i > 0)
                    else:
                        p2p.apply(src, dst, chain=i > 0)
                    src = dst
                last[0] = src
        else:
            slab = SlabSweep(U, kernels=CudaSlabKernels(args.mode))
            if world == 1:
                per_launch_sites = lat.volume
            else:
                per_launch_sites = max(ntl - 2, 0) * lat.slice_sites
            launches_per_app = slab.launches_per_apply(chained=True)  # steady state: the halo pack is fused
            extra_launches = slab.launches_per_apply(chained=False) - launches_per_app  # first application's pack

            def run_step(record=False):
                src = v0
                for i in range(apps):
                    dst = va if i % 2 == 0 else vb
                    slab.apply(src, dst, timer=(lambda: _EventTimer(stream, dominant_events)) if record else None,
                               chain=i > 0)
                    src = dst
                last[0] = src

        def step(record=False):
            run_step(record)

        bytes_per_launch = per_launch_sites * NN_BYTES[args.dtype]

        def parity_fn():
            """One step of the timed path (all `apps` chained applications from v0), against the C oracle
            iterated as many times on every rank's slab (halo faces from the neighbour ranks)."""
            from oracle import coracle

            run_step()
            if args.halo == "p2p":
                p2p.check()
            torch.cuda.synchronize(dev)
            U_h, want, got = U.numpy(), v0.numpy(), last[0].numpy()
            F = lat.slice_sites
            for _ in range(apps):
                if world == 1:
                    want = coracle.nn_sweep(U_h, want, lat.dims)
                else:
                    w_last = coracle.routine("mult_adj_su3_mat_vec", U_h[-F:, 3], want[-F:])
                    v_hi, w_lo = _exchange_faces(want[:F], w_last, rank, world, dev)
                    want = coracle.nn_sweep_slab(U_h, want, lat.dims, v_hi, w_lo)
            return got, want, (f"one timed step ({apps} chained applications from the step's input) on every "
                               f"rank's full {'x'.join(map(str, lat.dims))} slab, vs the C oracle iterated "
                               f"({'periodic sweep' if world == 1 else 'slab with the neighbours halo faces'})")

        launches_per_step = apps * launches_per_app + extra_launches
        sites_per_step = lat.volume * apps  # per rank
        del U_aos
    elif cfg["kind"] == "dslash":
        lat = Lattice4D(*cfg["global_dims"])  # replicas: every rank runs its own lattice
        U_aos = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen)
        U = Field.from_aos(lat, "mat4", U_aos)
        del U_aos
        v = Field.from_aos(lat, "vec", inputs.random_vectors_torch(lat.volume, None, tdt, dev, gen))
        if args.layout == "eo":  # checkerboarded fields: su3g_dslash_eo
            U, v = U.to_eo(), v.to_eo()
            torch.cuda.synchronize(dev)
        dout = v.empty_like()
        bytes_per_launch = lat.volume * DSLASH_BYTES[args.dtype]
        mode = args.mode

        def step(record=False):
            for parity in (0, 1):
                if record:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                sweeps.dslash(U, v, parity, out=dout, mode=mode)
                if record:
                    e1.record(stream)
                    dominant_events.append((e0, e1))

        def parity_fn():
            from oracle import coracle

            step()
            torch.cuda.synchronize(dev)
            want = coracle.nn_sweep(U.numpy(), v.numpy(), lat.dims)
            return dout.numpy(), want, "both parities of one timed step (D = D_eo + D_oe) vs the C oracle NN sweep"

        launches_per_step = 2
        sites_per_step = lat.volume
        cfg["name"] += f", {mode} arithmetic, {'checkerboarded (eo)' if args.layout == 'eo' else 't-sliced SoA'} fields"
    elif cfg["kind"] == "link":
        lat = Lattice4D(*cfg["global_dims"])
        if world > 1:
            raise SystemExit("the link-product workload is single-GPU (replicas only)")
        U_aos = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen)
        U = Field.from_aos(lat, "mat4", U_aos)
        del U_aos
        acc = Field(lat, "mat", tdt, dev)
        bytes_per_launch = lat.volume * LINK_BYTES[args.dtype]
        mode = args.mode

        def step(record=False):
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            sweeps.link_product(U, 1.0 / 6.0, mode=mode, out=acc)
            if record:
                e1.record(stream)
                dominant_events.append((e0, e1))

        def parity_fn():
            from oracle import coracle

            step()
            torch.cuda.synchronize(dev)
            want = coracle.link_product(U.numpy(), lat.dims, 1.0 / 6.0)
            return acc.numpy(), want, "the accumulator of one timed step at full size vs the C oracle link product"

        launches_per_step = 1
        sites_per_step = lat.volume
        cfg["name"] += f", {mode} arithmetic"
    else:  # routine streaming batch
        r = cfg["routine"]
        n = cfg["nsites"]
        rin, rout = ROUTINE_REALS[r]
        from paper_1309_0551_b200 import _lib
        from paper_1309_0551_b200 import types as T

        ins, _ = ROUTINE_LAYOUT[r]
        sfx = args.dtype
        esz = 4 if sfx == "f32" else 8
        set_bytes = n * (rin + rout) * esz
        bytes_per_launch = set_bytes
        # small configs (BASELINE configs[0]/[1]) take less than a launch: replay a CUDA graph of
        # R launches over R rotating operand sets totalling >= 2x L2, so every launch reads from HBM
        graph_mode = n < (1 << 20)
        R = 1
        if graph_mode:
            l2 = int(_lib.load().su3g_device_l2_bytes()) or (126 << 20)
            R = max(16, -(-2 * l2 // set_bytes))
        bufs = [torch.randn(R * n * k, dtype=tdt, device=dev, generator=gen) for k in ins]
        c = torch.empty(R * n * rout, dtype=tdt, device=dev)

        def launch(i=0):
            st = torch.cuda.current_stream(dev).cuda_stream
            p = [b.data_ptr() + i * n * k * esz for b, k in zip(bufs, ins)]
            pc = c.data_ptr() + i * n * rout * esz
            if r in SMADD_ROUTINES:
                _lib.call(f"su3g_{r}_{sfx}", p[0], p[1], 0.5, None, pc, n, st)
            elif r == "mult_adj_su3_mat_4vec":  # four separate destinations
                _lib.call(f"su3g_{r}_{sfx}", p[0], p[1], *(pc + d * n * 6 * esz for d in range(4)), n, st)
            elif r == "sub_four_su3_vecs":  # in place on the first operand
                _lib.call(f"su3g_{r}_{sfx}", *p, n, st)
            else:
                _lib.call(f"su3g_{r}_{sfx}", p[0], p[1], pc, n, st)

        graph = None
        if graph_mode:
            for i in range(2):
                launch(i)  # warm the launch caches before capture
            torch.cuda.synchronize(dev)
            graph = torch.cuda.CUDAGraph()
            # the R launches are independent batch calls: the graph forks them over args.streams
            # branches so that several small batches are in flight at once (1 = one serial chain)
            C = max(1, min(args.streams, R))
            side = [torch.cuda.Stream(dev) for _ in range(C)] if C > 1 else []
            with torch.cuda.graph(graph):
                if C == 1:
                    for i in range(R):
                        launch(i)
                else:
                    cap = torch.cuda.current_stream(dev)
                    for sb in side:
                        sb.wait_stream(cap)
                    for i in range(R):
                        with torch.cuda.stream(side[i % C]):
                            launch(i)
                    for sb in side:
                        cap.wait_stream(sb)
            cfg["name"] = (f"{r} on {n} sites (BASELINE configs[{0 if n <= 4096 else 1}] size), CUDA graph of {R} "
                           f"launches over rotating operand sets (> 2x L2), {C} concurrent branch{'es' if C > 1 else ''}")
            cfg["graph_branches"] = C

        def step(record=False):
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                launch()
            if record:
                e1.record(stream)
                dominant_events.append((e0, e1))

        def parity_fn():
            """Operand set 0 through the same launch, against the oracle (first 2^20 sites)."""
            from oracle import coracle
            from oracle import routines as OR

            m = min(n, 1 << 20)
            spec_ = T.routine_spec(r)
            shapes = [T.OPERAND_SHAPES[k] for k in spec_.operands if k != "scalar"]
            before = [b[: n * k].view((n,) + sh)[:m].cpu().numpy() for b, k, sh in zip(bufs, ins, shapes)]
            launch(0)
            torch.cuda.synchronize(dev)
            if r == "sub_four_su3_vecs":
                got = bufs[0][: n * 6].view(n, 3, 2)[:m].cpu().numpy()
            elif r == "mult_adj_su3_mat_4vec":
                got = np.stack([c[d * n * 6 : (d + 1) * n * 6].view(n, 3, 2)[:m].cpu().numpy() for d in range(4)], 1)
            else:
                got = c[: n * rout].view((n,) + T.OPERAND_SHAPES[spec_.result])[:m].cpu().numpy()
            ops = before[:2] + [before[0].dtype.type(0.5)] if r in SMADD_ROUTINES else before
            if r in coracle.ROUTINE_IDS:
                want = coracle.routine(r, *ops)
            else:
                want = OR.ALL_ROUTINES[r](*ops)
            return got, want, f"operand set 0 of the timed launch ({m} sites) vs the oracle"

        launches_per_step = R
        sites_per_step = n * R
        launches_per_event = R  # one timed event brackets R graph-replayed launches

    # ---- warm-up, then the timed region ---------------------------------
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    dispatched = _l.last_kernel()  # the kernel the last launch of a step dispatched to
    if cfg["kind"] == "nn" and args.halo == "p2p":
        dispatched = "k_p2p_boundary + interior " + dispatched + " (timed together, per application)"
    elif cfg["kind"] == "nn" and world > 1:
        dispatched = "interior: " + _interior_kernel(sweeps, U, v0, vb, lat.nt, args.mode)
    clocks = ClockSampler(local)
    barrier(world, dev)
    torch.cuda.synchronize(dev)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.stop()
    barrier(world, dev)
    elapsed_ms = max_over_ranks(t0.elapsed_time(t1), world, dev)
    kern_ms = [a.elapsed_time(b) for a, b in dominant_events]
    kern_avg_ms = max_over_ranks(float(np.mean(kern_ms)) / launches_per_event if kern_ms else float("nan"), world, dev)

    total_sites = sites_per_step * world * args.steps
    value = total_sites / (elapsed_ms / 1e3)
    peak, peak_src = peak_hbm()
    achieved = bytes_per_launch / (kern_avg_ms / 1e3) / 1e9 if kern_ms else None
    from paper_1309_0551_b200 import flops as _flops

    intensity = _flops.intensity(cfg["routine"] if cfg["kind"] == "routine" else cfg["kind"], args.dtype)

    if cfg["kind"] == "nn" and args.halo == "p2p":
        p2p.check()  # a timed-out halo wait voids the run

    # ---- parity (the checker, outside the timed region) ----------------------
    parity = None
    if not args.no_parity:
        parity = _parity(parity_fn, args, cfg, world, dev)

    # ---- e2e through the host-buffer path ---------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, cfg, rank, world, dev, tdt, stream)

    # ---- the N > 1 per-rank schedule, run on this one GPU ---------------------
    slab_probe = None
    if cfg["kind"] == "nn" and world == 1 and args.halo == "nccl" and not args.no_slab_probe:
        slab_probe = _slab_schedule_probe(U, v0, va, vb, cfg["apps"], args, stream, value, elapsed_ms)

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if args.workload == "nn-weak" else ("strong" if args.workload == "nn-strong" else "weak"),
        "vs_baseline": None,
        "dtype": args.dtype,
        "arithmetic": args.mode if cfg["kind"] in ("nn", "link", "dslash") else "exact",
        "data": "synthetic (seeded SU(3) Gram-Schmidt links + complex-Gaussian vectors, generated on device)",
        "config": {
            "workload": cfg["name"],
            "lattice": list(cfg.get("global_dims", [])) or None,
            "sites_per_gpu": sites_per_step // max(cfg["apps"], 1),
            "applications_per_step": cfg["apps"],
            "parallelism": (f"t-slab x{world}, halos via " + ("fused NVLink push (p2p)" if args.halo == "p2p" else "NCCL")
                            if cfg["kind"] == "nn" else f"replicas x{world}"),
            "l2": "inputs larger than L2 (U alone > 1 GB/GPU); no flush needed",
        },
        "impl": "b200",
        "hbm_gbs": achieved,
        "roofline": {
            "bound": "hbm",
            "kernel": dispatched,
            "achieved": achieved,
            "peak": peak,
            "peak_source": peak_src,
            "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None,
            "peak_datasheet": DATASHEET_HBM_GBS,
            "frac_datasheet": (achieved / DATASHEET_HBM_GBS) if achieved else None,
            "traffic": traffic_for(args.workload, args.dtype, args.mode, dispatched),
            "algorithmic_bytes_per_launch": bytes_per_launch,
            "kernel_avg_ms": kern_avg_ms,
            "compute_floor": _compute_floor(cfg, args, bytes_per_launch, kern_avg_ms, dispatched),
        },
        "flops_per_site": intensity["flops_per_site"],
        "ai_flop_per_byte": intensity["ai_flop_per_byte"],
        "parity": parity,
        "gpu_launches": launches_per_step * args.steps,
        "launches_per_step": launches_per_step,
        "clocks": clocks.summary(),
        "e2e": e2e,
    }
    if slab_probe is not None:
        line["slab_schedule_1gpu"] = slab_probe
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args, cfg)
    return line


def _slab_schedule_probe(U, v0, va, vb, apps, args, stream, value, elapsed_ms):
    """The per-rank schedule of an N > 1 t-slab run, timed on this one GPU against itself.

    A one-rank NCCL communicator sends the two halo faces to itself (su3g_slab_nn_sweep: halo pack,
    grouped send/recv on the communicator's stream, the interior slices with 4 SMs left free for
    NCCL's kernels, then both boundary slices in one launch) -- every launch and every SM
    reservation of a multi-GPU rank, minus the NVLink transfer itself, which overlaps the interior.
    Reported beside `value` as a predictor of the weak-scaling efficiency; it is NOT a multi-GPU
    measurement (only one GPU is available here)."""
    import torch

    from paper_1309_0551_b200 import _lib as _l
    from paper_1309_0551_b200.comm import NativeComm, native_slab_sweep

    if U.lattice.nt < 3:
        return None
    saved = 0
    _l.set_option("sm_reserve", 4)
    try:
        with NativeComm(1, 0, NativeComm.unique_id()) as comm:
            def step():
                src = v0
                for i in range(apps):
                    dst = va if i % 2 == 0 else vb
                    native_slab_sweep(comm, U, src, dst, args.mode)
                    src = dst

            for _ in range(max(args.warmup, 3)):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            comm.check()
            ms = e0.elapsed_time(e1)
    finally:
        _l.set_option("sm_reserve", saved)
    sites = U.lattice.volume * apps * args.steps
    probe_value = sites / (ms / 1e3)
    return {
        "value": probe_value, "unit": UNIT, "ms_per_step": ms / args.steps,
        "vs_periodic_value": probe_value / value,
        "what": "one GPU running the per-rank schedule of an N>1 t-slab run against a one-rank NCCL communicator "
                "(self send/recv of both halo faces, halo pack, interior with 4 SMs reserved, fused boundary "
                "launch); predicts the per-GPU rate at N>1 minus the NVLink transfer, which overlaps the interior. "
                "Not a multi-GPU measurement.",
    }


def _exchange_faces(v_first, w_last, rank, world, dev):
    """Parity check at N > 1: v on this rank's first slice goes to rank r-1, the oracle's w on its
    last slice to rank r+1 (the t-slab halos); returns (v_hi, w_lo) as numpy."""
    import torch
    import torch.distributed as dist

    sv = torch.from_numpy(np.ascontiguousarray(v_first)).to(dev)
    sw = torch.from_numpy(np.ascontiguousarray(w_last)).to(dev)
    v_hi, w_lo = torch.empty_like(sv), torch.empty_like(sw)
    up, dn = (rank + 1) % world, (rank - 1) % world
    ops = [dist.P2POp(dist.isend, sv, dn), dist.P2POp(dist.irecv, v_hi, up),
           dist.P2POp(dist.isend, sw, up), dist.P2POp(dist.irecv, w_lo, dn)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    torch.cuda.synchronize(dev)
    return v_hi.cpu().numpy(), w_lo.cpu().numpy()


def _parity(parity_fn, args, cfg, world, dev):
    """Run the workload's parity check on every rank; rank 0 reports the worst."""
    from oracle.compare import parity_record

    got, want, what = parity_fn()
    exact = not (cfg["kind"] in ("nn", "link", "dslash") and args.mode == "fma")
    rec = parity_record(got, want, exact, what)
    del got, want
    if world > 1:
        rec["max_floored_rel_err"] = max_over_ranks(rec["max_floored_rel_err"], world, dev)
        rec["bitwise"] = max_over_ranks(0.0 if rec["bitwise"] else 1.0, world, dev) == 0.0
        rec["pass"] = max_over_ranks(0.0 if rec["pass"] else 1.0, world, dev) == 0.0
        rec["ranks_checked"] = world
    return rec


class _EventTimer:
    """CUDA events around one kernel launch on `stream` (the dominant kernel's duration)."""

    def __init__(self, stream, sink):
        import torch

        self.stream, self.sink = stream, sink
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.e0.record(self.stream)
        return self

    def __exit__(self, *exc):
        self.e1.record(self.stream)
        self.sink.append((self.e0, self.e1))
        return False


def _interior_kernel(sweeps, U, va, vb, nt, mode) -> str:
    """Name of the kernel the interior slices of a t-slab dispatch to (the dominant launch at N > 1)."""
    import torch

    from paper_1309_0551_b200 import _lib

    if nt <= 2:
        return "none (every slice is a boundary slice)"
    sweeps.nn_sweep(U, va, out=vb, t_range=(1, nt - 1), mode=mode)
    torch.cuda.synchronize()
    return _lib.last_kernel()


def _pipelined_e2e(hosts, out_host, compute, steps, world, dev, stream):
    """Time `steps` end-to-end steps, pipelined across steps without skipping any copy: step i+1's
    inputs stream host->device on a copy-in stream while step i computes, and step i's result leaves
    device->host on a third stream (PCIe is full duplex).  Double-buffered device staging; events
    order buffer reuse.  compute(dev_inputs, dev_out) enqueues the step's work on `stream`.
    Returns the elapsed milliseconds (max over ranks)."""
    import torch

    cin, cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    d_in = [[torch.empty_like(h, device=dev) for h in hosts] for _ in range(2)]
    d_out = [torch.empty_like(out_host, device=dev) for _ in range(2)]
    outs_h = [out_host, torch.empty_like(out_host).pin_memory()]
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("h2d", "comp", "d2h")}

    def enqueue(i):
        b = i % 2
        with torch.cuda.stream(cin):
            if i >= 2:
                cin.wait_event(ev["comp"][b])  # step i-2 has finished reading this input buffer
            for d, h in zip(d_in[b], hosts):
                d.copy_(h, non_blocking=True)
            ev["h2d"][b].record(cin)
        stream.wait_event(ev["h2d"][b])
        if i >= 2:
            stream.wait_event(ev["d2h"][b])  # step i-2's result has left this output buffer
        compute(d_in[b], d_out[b])
        ev["comp"][b].record(stream)
        with torch.cuda.stream(cout):
            cout.wait_event(ev["comp"][b])
            outs_h[b].copy_(d_out[b], non_blocking=True)
            ev["d2h"][b].record(cout)

    for i in range(3):  # warm-up
        enqueue(i)
    torch.cuda.synchronize(dev)
    barrier(world, dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cin)
    stream.wait_event(e0)
    for i in range(steps):
        enqueue(i)
    for b in range(2):
        stream.wait_event(ev["d2h"][b])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier(world, dev)
    return max_over_ranks(e0.elapsed_time(e1), world, dev)


def _sequential_e2e(hosts, out_host, compute, steps, world, dev, stream):
    """The same steps on one stream, copy-in -> compute -> copy-out: for small steps, where the
    host cost of the pipelined form's extra streams and events outweighs the overlap."""
    import torch

    d_in = [torch.empty_like(h, device=dev) for h in hosts]
    d_out = torch.empty_like(out_host, device=dev)

    def step():
        for d, h in zip(d_in, hosts):
            d.copy_(h, non_blocking=True)
        compute(d_in, d_out)
        out_host.copy_(d_out, non_blocking=True)

    for _ in range(3):
        step()
    torch.cuda.synchronize(dev)
    barrier(world, dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier(world, dev)
    return max_over_ranks(e0.elapsed_time(e1), world, dev)


def measure_e2e(args, cfg, rank, world, dev, tdt, stream):
    """Same metric through the reference-facing path: pinned host AoS in, host AoS out, copies timed."""
    import torch

    from paper_1309_0551_b200 import inputs, sweeps
    from paper_1309_0551_b200.lattice import Field, Lattice4D
    from paper_1309_0551_b200.slab import CudaSlabKernels, SlabSweep

    steps = max(3, min(args.steps, 10))
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + rank)
    path = ("pinned host AoS -> H2D (copy stream, overlapping the previous step) -> {} -> D2H (its own stream)")
    if cfg["kind"] == "nn":
        lat = Lattice4D(*cfg["global_dims"]).slab(world, rank)
        U_h = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen).cpu().pin_memory()
        v_h = inputs.random_vectors_torch(lat.volume, None, tdt, dev, gen).cpu().pin_memory()
        out_h = torch.empty_like(v_h).pin_memory()
        Uf = Field(lat, "mat4", tdt, dev)
        va, vb = Field(lat, "vec", tdt, dev), Field(lat, "vec", tdt, dev)
        if args.halo == "p2p":
            from paper_1309_0551_b200.p2p import P2PSlabSweep

            slab = P2PSlabSweep(Uf, mode=args.mode)

            def run_apps(a, b, n):
                return slab.apply_n(a, n, scratch=b)
        else:
            slab = SlabSweep(Uf, kernels=CudaSlabKernels(args.mode))

            def run_apps(a, b, n):
                return slab.apply_n(a, b, n)

        def compute(d_in, d_out):
            Field.from_aos(lat, "mat4", d_in[0], out=Uf)
            Field.from_aos(lat, "vec", d_in[1], out=va)
            run_apps(va, vb, cfg["apps"]).to_aos(out=d_out)

        hosts, sites = [U_h, v_h], lat.volume * cfg["apps"]
        what = "AoS->SoA -> kernels (+halos) -> SoA->AoS"
    elif cfg["kind"] == "dslash":
        lat = Lattice4D(*cfg["global_dims"])
        U_h = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen).cpu().pin_memory()
        v_h = inputs.random_vectors_torch(lat.volume, None, tdt, dev, gen).cpu().pin_memory()
        out_h = torch.empty_like(v_h).pin_memory()
        Uf, vf = Field(lat, "mat4", tdt, dev), Field(lat, "vec", tdt, dev)
        of = vf.empty_like()
        eo = args.layout == "eo"
        if eo:
            Ue, ve = Field(lat, "mat4", tdt, dev, layout="eo"), Field(lat, "vec", tdt, dev, layout="eo")
            oe = ve.empty_like()

        def compute(d_in, d_out):
            Field.from_aos(lat, "mat4", d_in[0], out=Uf)
            Field.from_aos(lat, "vec", d_in[1], out=vf)
            if eo:
                Uf.to_eo(out=Ue)
                vf.to_eo(out=ve)
                for parity in (0, 1):
                    sweeps.dslash(Ue, ve, parity, out=oe, mode=args.mode)
                oe.to_soa(out=of)
            else:
                for parity in (0, 1):
                    sweeps.dslash(Uf, vf, parity, out=of, mode=args.mode)
            of.to_aos(out=d_out)

        hosts, sites = [U_h, v_h], lat.volume
        what = "AoS->SoA" + (" -> eo" if eo else "") + " -> both parities -> SoA->AoS"
    elif cfg["kind"] == "link":
        lat = Lattice4D(*cfg["global_dims"])
        U_h = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen).cpu().pin_memory()
        out_h = torch.empty((lat.volume, 3, 3, 2), dtype=tdt).pin_memory()
        Uf = Field(lat, "mat4", tdt, dev)
        acc = Field(lat, "mat", tdt, dev)

        def compute(d_in, d_out):
            Field.from_aos(lat, "mat4", d_in[0], out=Uf)
            sweeps.link_product(Uf, 1.0 / 6.0, mode=args.mode, out=acc).to_aos(out=d_out)

        hosts, sites = [U_h], lat.volume
        what = "AoS->SoA -> link product -> SoA->AoS"
    else:
        from paper_1309_0551_b200 import kernels
        from paper_1309_0551_b200 import types as T

        r = cfg["routine"]
        n = cfg["nsites"]
        gen_c = torch.Generator(device=dev)
        gen_c.manual_seed(99)
        spec = T.routine_spec(r)
        kinds = [k for k in spec.operands if k != "scalar"]
        hosts = [torch.randn((n,) + T.OPERAND_SHAPES[k], dtype=tdt, generator=gen_c, device=dev).cpu().pin_memory()
                 for k in kinds]
        out_h = torch.empty((n,) + T.OPERAND_SHAPES[spec.result], dtype=tdt).pin_memory()
        fn = kernels.KERNELS[r]

        def compute(d_in, d_out):
            if r in SMADD_ROUTINES:
                fn(d_in[0], d_in[1], 0.5, out=d_out)
            elif r == "mult_adj_su3_mat_4vec":
                fn(d_in[0], d_in[1], outs=[d_out[:, d] for d in range(4)])  # strided views: staged + copied
            elif r == "sub_four_su3_vecs":
                d_out.copy_(fn(*d_in))  # in place on its first operand
            else:
                fn(d_in[0], d_in[1], out=d_out)

        sites = n
        what = "drop-in routine (AoS, C ABI)"
    step_bytes = sum(h.numel() * h.element_size() for h in hosts) + out_h.numel() * out_h.element_size()
    if step_bytes >= (4 << 20):  # copies long enough to hide behind each other (65536-site routines: +13%)
        ms = _pipelined_e2e(hosts, out_h, compute, steps, world, dev, stream)
    else:
        ms = _sequential_e2e(hosts, out_h, compute, steps, world, dev, stream)
        path = path.replace(" (copy stream, overlapping the previous step)", "").replace(" (its own stream)", "")
    return {
        "value": sites * world * steps / (ms / 1e3),
        "unit": UNIT,
        "h2d_bytes_per_step": int(sum(h.numel() * h.element_size() for h in hosts)),
        "d2h_bytes_per_step": int(out_h.numel() * out_h.element_size()),
        "steps": steps,
        "path": path.format(what),
    }


# ----------------------------------------------------------------------------
# CPU side: the reference's own implementation of the path on host cores
# ----------------------------------------------------------------------------
#
# The reference (su3bench) is pure Python + numpy.  It is installed offline into the git-ignored
# baseline/_ref/ (__graft_entry__.build(); it travels to the GPU box with the snapshot) and driven
# through its own public API: SiteBuffer for the fields, simd routines for the arithmetic, and
# bench.run for the per-routine streaming rows (bench.py:229-271).  The sweeps have no reference
# function; they are the composition of the reference's routines fixed by SURVEY.md 8(c).  When
# baseline/_ref is missing, the numpy restatement in oracle/ (bit-identical to su3bench, pinned by
# tests/test_oracle_golden.py) stands in and the record says kind "port".

REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def _su3bench():
    """The installed reference package, or None."""
    if not os.path.isdir(os.path.join(REF_PATH, "su3bench")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        import su3bench.bench  # noqa: F401
        import su3bench.lattice  # noqa: F401
        import su3bench.simd  # noqa: F401

        return sys.modules["su3bench"]
    except Exception:  # noqa: BLE001
        return None


def _host_info() -> dict:
    """CPU model and numpy version of the host the CPU baseline ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "numpy": np.__version__, "host_cpus": os.cpu_count()}


class _Pinned:
    """Pin the process to one CPU for the timed region, as the reference's bench does (bench.py:134-152)."""

    def __enter__(self):
        self.prev = None
        try:
            self.prev = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(self.prev)})
        except (AttributeError, OSError):
            self.prev = None
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            try:
                os.sched_setaffinity(0, self.prev)
            except OSError:
                pass
        return False


class RefSweep:
    """The composed reference sweep on output t-slices [t0, t0+k) of the workload's full lattice.

    Fields live in the reference's own SiteBuffer (randomize: the reference's uniform draw; timing does
    not depend on values).  Each output slice is computed exactly once per call: x, y, z shifts are
    periodic rolls inside the window, t neighbours come from the slices on either side, so a sample of
    k slices is k x F site-ops of the real workload (SURVEY.md 8(c) association).
    """

    def __init__(self, cfg, dtype: str):
        self.kind = cfg["kind"]
        self.dims = cfg["global_dims"]
        prec = "single" if dtype == "f32" else "double"
        ref = _su3bench()
        fields = {"U": "mat4"} if self.kind == "link" else {"U": "mat4", "v": "vec"}
        if ref is not None:
            from su3bench import simd
            from su3bench.lattice import Lattice4D as RLat
            from su3bench.lattice import SiteBuffer

            buf = SiteBuffer(RLat(*self.dims), fields, precision=prec)
            buf.randomize(12345)
            self.U = buf["U"]
            self.v = buf["v"] if "v" in fields else None
            self.ops = simd
            self.source = "reference"
            self.impl = "su3bench (baseline/_ref): SiteBuffer + simd routines, composed as SURVEY.md 8(c)"
        else:
            from oracle import routines as R
            from oracle import sitebuffer as OS

            V = int(np.prod(self.dims))
            f = OS.randomize(V, fields, np.float32 if dtype == "f32" else np.float64, 12345)
            self.U, self.v = f["U"], f.get("v")
            self.ops = R
            self.source = "port"
            self.impl = "numpy restatement in oracle/ (bit-identical to su3bench), composed as SURVEY.md 8(c)"
        nx, ny, nz, nt = self.dims
        self.F = nx * ny * nz
        self.s = self.U.dtype.type(1.0 / 6.0)

    def _sh(self, f, k, mu, step):
        nx, ny, nz, _ = self.dims
        g = f.reshape((k, nz, ny, nx) + f.shape[1:])
        return np.roll(g, -step, axis=3 - mu).reshape(f.shape)

    def _slices(self, f, t, k):
        nt, F = self.dims[3], self.F
        if t + k <= nt and t >= 0:
            return f[t * F : (t + k) * F]
        return np.concatenate([f[((t + j) % nt) * F : ((t + j) % nt + 1) * F] for j in range(k)])

    def __call__(self, t0: int, k: int):
        o, F = self.ops, self.F
        Uw = self._slices(self.U, t0, k)
        if self.kind == "link":
            Unext = self._slices(self.U, t0 + 1, k)
            acc = np.zeros((k * F, 3, 3, 2), dtype=self.U.dtype)
            for mu, nu in ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)):
                b = self._sh(Uw[:, nu], k, mu, +1)
                c = self._sh(Uw[:, mu], k, nu, +1) if nu < 3 else Unext[:, mu]
                acc = o.scalar_mult_add_su3_matrix(acc, o.mult_su3_na(o.mult_su3_nn(Uw[:, mu], b), c), self.s)
            return acc
        vw = self._slices(self.v, t0, k)
        fw = [o.mult_su3_mat_vec(Uw[:, mu], self._sh(vw, k, mu, +1)) for mu in range(3)]
        fw.append(o.mult_su3_mat_vec(Uw[:, 3], self._slices(self.v, t0 + 1, k)))
        bw = [o.mult_adj_su3_mat_vec(self._sh(Uw[:, mu], k, mu, -1), self._sh(vw, k, mu, -1)) for mu in range(3)]
        bw.append(o.mult_adj_su3_mat_vec(self._slices(self.U, t0 - 1, k)[:, 3], self._slices(self.v, t0 - 1, k)))
        acc = o.add_su3_vector(o.add_su3_vector(o.add_su3_vector(fw[0], fw[1]), fw[2]), fw[3])
        return o.sub_four_su3_vecs(acc, bw[0], bw[1], bw[2], bw[3])


def _sample_slices(cfg) -> int:
    """t-slices per timed call: about 1-3 s of single-core work on the full-size workloads."""
    nx, ny, nz, nt = cfg["global_dims"]
    per_slice = nx * ny * nz * (8 if cfg["kind"] == "link" else 1)
    k = max(1, min(nt, (1 << 19) // max(per_slice, 1)))
    while nt % k:
        k -= 1
    return k


def _ref_routine_rate(cfg, dtype: str, budget_s: float):
    """Per-routine streaming rows through su3bench.bench.run (backend 'vector', bench.py:229-271)."""
    ref = _su3bench()
    prec = "single" if dtype == "f32" else "double"
    n = min(cfg["nsites"], 1 << 16)
    dims = {4096: (8, 8, 8, 8), 65536: (16, 16, 16, 16)}.get(n, (16, 16, 16, 16))
    V = int(np.prod(dims))
    if ref is not None:
        from su3bench.bench import BenchConfig, run

        rec = run(BenchConfig(routine=cfg["routine"], backend="vector", precision=prec, mode="streaming", dims=dims,
                              repetitions=1, warmup=3, min_region_s=budget_s))
        return rec.invocations, rec.elapsed_s, "reference", (
            f"su3bench.bench.run(BenchConfig(routine={cfg['routine']!r}, backend='vector', mode='streaming', "
            f"dims={dims})) -- the reference's own streaming timer, pinned to one CPU")
    from oracle import routines as R
    from paper_1309_0551_b200 import types as T

    rng = np.random.default_rng(12345)
    dt = np.float32 if dtype == "f32" else np.float64
    spec = T.routine_spec(cfg["routine"])
    ops = [dt(0.5) if k == "scalar" else rng.uniform(-1, 1, (V,) + T.OPERAND_SHAPES[k]).astype(dt) for k in spec.operands]
    fn = R.ALL_ROUTINES[cfg["routine"]]
    with _Pinned():
        fn(*ops)
        n_calls, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s:
            fn(*ops)
            n_calls += 1
        el = time.perf_counter() - t0
    return n_calls * V, el, "port", f"numpy restatement of {cfg['routine']} on {dims} ({V} sites), one CPU"


def cpu_baseline(args, cfg, budget_s=12.0):
    """The b200 line's cpu_baseline: the reference on one pinned core over a bounded sample (N=1, rank 0)."""
    if cfg["kind"] == "routine":
        ops, el, kind, desc = _ref_routine_rate(cfg, args.dtype, budget_s / 3)
        return {"value": ops / el, "unit": UNIT, "cores": 1, "kind": kind, "sample": desc, **_host_info()}
    rs = RefSweep(cfg, args.dtype)
    k = _sample_slices(cfg)
    nt = cfg["global_dims"][3]
    with _Pinned():
        rs(0, k)  # warm
        n, t = 0, time.perf_counter()
        while True:
            rs((n * k) % nt, k)
            n += 1
            el = time.perf_counter() - t
            if el >= budget_s or n >= 50:
                break
    sites = n * k * rs.F
    return {
        "value": sites / el, "unit": UNIT, "cores": 1, "kind": rs.source,
        "sample": (f"{rs.impl}; {n} calls of {k} output t-slice(s) each ({sites} site-ops) of the full "
                   f"{'x'.join(map(str, cfg['global_dims']))} lattice in {el:.2f} s, one pinned CPU"),
        **_host_info(),
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on this box's host cores, on the b200 arm's
    workload and metric.  Rank 0 alone runs it (the other ranks exit without work)."""
    cfg = workload_config(args, world)
    if rank != 0:
        return None
    if cfg["kind"] == "routine":
        budget = max(0.05, 20.0 / max(args.steps + args.warmup, 1))
        tot_ops, tot_el = 0, 0.0
        for i in range(args.warmup + args.steps):
            ops, el, kind, desc = _ref_routine_rate(cfg, args.dtype, budget)
            if i >= args.warmup:
                tot_ops += ops
                tot_el += el
        value, el = tot_ops / tot_el, tot_el
        sample, upper = desc + f"; {args.steps} timed calls", None
    else:
        rs = RefSweep(cfg, args.dtype)
        kind = rs.source
        k = _sample_slices(cfg)
        nt = cfg["global_dims"][3]
        with _Pinned():
            for i in range(args.warmup):
                rs((i * k) % nt, k)
            t0 = time.perf_counter()
            for i in range(args.steps):
                rs((i * k) % nt, k)
            el = time.perf_counter() - t0
        value = args.steps * k * rs.F / el
        sample = (f"{rs.impl}; each step = {k} output t-slice(s) ({k * rs.F} site-ops) of the full "
                  f"{'x'.join(map(str, cfg['global_dims']))} lattice, windows cycling over t; one pinned CPU "
                  f"(the reference is single-threaded numpy)")
        upper = _upper_bound_aggregate(rs, cfg)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": el * 1e3 / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if args.workload == "nn-weak" else ("strong" if args.workload == "nn-strong" else "weak"),
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (the reference's SiteBuffer.randomize uniform fields; timing is value-independent)",
        "config": {"workload": cfg["name"], "lattice": list(cfg.get("global_dims", [])) or None,
                   "same_config": not args.dims},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample, **_host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if upper is not None:
        line["upper_bound_aggregate"] = upper
    return line


def _upper_bound_aggregate(rs, cfg, max_s=20.0):
    """All host threads on disjoint t-windows at once -- labelled an upper bound, NOT the reference
    (which is one single-threaded process); numpy releases the GIL inside its loops."""
    from concurrent.futures import ThreadPoolExecutor

    threads = os.cpu_count() or 1
    nt = cfg["global_dims"][3]
    k = _sample_slices(cfg)
    windows = [(t, k) for t in range(0, nt, k)]
    if len(windows) < threads:
        k1 = max(1, nt // threads)
        while nt % k1:
            k1 -= 1
        windows = [(t, k1) for t in range(0, nt, k1)]
    with ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        done = 0
        for _ in ex.map(lambda w: rs(*w), windows):
            done += 1
            if time.perf_counter() - t0 > max_s:
                break
        el = time.perf_counter() - t0
    sites = sum(w[1] for w in windows[:done]) * rs.F
    return {"value": sites / el, "unit": UNIT, "threads": threads, "kind": rs.source,
            "label": "upper bound: all host threads on disjoint t-windows of one lattice pass; not the reference's "
                     "configuration (single-threaded)"}


def _spawn_ranks(args, argv) -> int:
    """--gpus N > 1 without a torch.distributed launcher: start the N ranks here (one process per GPU)
    with torch.distributed.run on 127.0.0.1, and return its exit code.  Rank 0 prints the line."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ, SU3G_BENCH_SPAWNED="1")
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    args = parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not os.environ.get("SU3G_BENCH_SPAWNED"):
        raise SystemExit(_spawn_ranks(args, argv))
    rank, world, local = init_dist(args)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_b200(args, rank, world, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
