"""t-slab domain decomposition of the NN sweep across GPUs (BASELINE configs[4]).

The global lattice nx*ny*nz*nt is cut along t into G equal slabs, one per
rank (one process per GPU, torch.distributed over NCCL).  A fixed-t slice is
a contiguous block of sites in the reference numbering (lattice.py:3-6), so a
rank's fields are contiguous sub-arrays and its t-faces are contiguous SoA
blocks.

Per application of D, rank r needs two one-site halos:
  * v on the first t-slice of rank r+1  (forward +t term of its last slice);
  * w = U_t(x)^dag v(x) on the last t-slice of rank r-1 (backward -t term of
    its first slice).  The owner computes w with the same arithmetic the
    unsharded kernel uses, so the sharded result is BIT-IDENTICAL to the
    single-GPU sweep; 6 reals cross the link per face site instead of 24.

Schedule per application (compute stream C, NCCL's stream N):
  C: pack w_last                        (su3g_nn_halo_w; skipped when chained, see below)
  N: send v_first -> r-1, recv v_hi <- r+1, send w_last -> r+1, recv w_lo <- r-1
  C: interior slices t in [1, nt_local-1)    -- overlaps the exchange
  C: wait(N); boundary slices t = 0 and t = nt_local-1 in one launch (su3g_nn_sweep_edges), which
     also packs w_last of its result for the next application
Chained applications (apply_n, or apply(..., chain=True) when v is the previous call's out) reuse
that packed w instead of launching the pack kernel again.

The compute is pluggable (``kernels``) so the exchange logic can be exercised
on CPU ranks over gloo in the tests; the product default is the CUDA kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import sweeps
from .lattice import Field

TAG_V = 11
TAG_W = 12
SM_RESERVE = 4  # SMs kept free for the NCCL halo-exchange kernels while the interior runs


class CudaSlabKernels:
    """Device compute for one slab: libsu3g kernels on t-sliced SoA fields."""

    def __init__(self, mode: str = "exact"):
        self.mode = mode

    def alloc_face(self, v: Field) -> torch.Tensor:
        return torch.empty((6, v.lattice.slice_sites), dtype=v.dtype, device=v.device)

    def first_face(self, v: Field) -> torch.Tensor:
        return v.face(0)

    def halo_w(self, U: Field, v: Field, w: torch.Tensor) -> None:
        sweeps.nn_halo_w(U, v, w, mode=self.mode)

    def sweep(self, U: Field, v: Field, out: Field, t_range, v_hi, w_lo) -> None:
        sweeps.nn_sweep(U, v, out=out, t_range=t_range, v_hi=v_hi, w_lo=w_lo, mode=self.mode)

    def edges(self, U: Field, v: Field, out: Field, v_hi, w_lo, w_next) -> None:
        """Both boundary slices in one launch; w_next <- w_last of out (the next application's halo)."""
        sweeps.nn_edges(U, v, out, v_hi=v_hi, w_lo=w_lo, w_next=w_next, mode=self.mode)

    def nt(self, v: Field) -> int:
        return v.lattice.nt

    def prepare(self, world: int) -> None:
        """Leave SMs free for NCCL's kernels so the halo exchange overlaps the interior sweep.

        The persistent sweep kernel fills every SM (all registers, ~210 KB smem), so a
        concurrently launched NCCL kernel could not be co-scheduled until it finished.
        """
        from . import _lib

        _lib.set_option("sm_reserve", SM_RESERVE if world > 1 else 0)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def _maybe(timer):
    return timer() if timer is not None else _Null()


def boundary_ranges(nt_local: int):
    """(interior range, boundary ranges) of local t-slices; halos only touch the boundary."""
    if nt_local <= 2:
        return None, [(t, t + 1) for t in range(nt_local)]
    return (1, nt_local - 1), [(0, 1), (nt_local - 1, nt_local)]


class SlabSweep:
    """Applies D on this rank's t-slab, exchanging halos with the t-neighbour ranks."""

    def __init__(self, U, kernels=None, group=None):
        self.U = U
        self.k = kernels if kernels is not None else CudaSlabKernels()
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self._faces = None
        self._w_of = None  # the Field whose w_last the face buffer holds (packed by the edges launch)
        if hasattr(self.k, "prepare"):
            self.k.prepare(self.world)

    @property
    def up(self) -> int:
        return (self.rank + 1) % self.world

    @property
    def down(self) -> int:
        return (self.rank - 1) % self.world

    def _buffers(self, v):
        if self._faces is None:
            self._faces = (self.k.alloc_face(v), self.k.alloc_face(v), self.k.alloc_face(v))
        return self._faces

    def _peer(self, r: int) -> int:
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def exchange(self, v, w_send, v_hi, w_lo):
        """Post the four halo transfers; returns the pending requests."""
        ops = [
            dist.P2POp(dist.isend, self.k.first_face(v), self._peer(self.down), self.group, TAG_V),
            dist.P2POp(dist.irecv, v_hi, self._peer(self.up), self.group, TAG_V),
            dist.P2POp(dist.isend, w_send, self._peer(self.up), self.group, TAG_W),
            dist.P2POp(dist.irecv, w_lo, self._peer(self.down), self.group, TAG_W),
        ]
        return dist.batch_isend_irecv(ops)

    def apply(self, v, out, timer=None, chain=False):
        """out = D v on this slab (periodic in t across the ranks).

        ``timer`` (optional) is a context-manager factory wrapped around the
        dominant kernel launch -- the whole sweep on one rank, the interior
        slices otherwise (bench.py records CUDA events with it).
        ``chain=True`` promises that v is the unmodified ``out`` of the previous
        call: its w_last was packed by that call's boundary launch.
        """
        if self.world == 1:
            with _maybe(timer):
                self.k.sweep(self.U, v, out, (0, self.k.nt(v)), None, None)
            return out
        w_send, v_hi, w_lo = self._buffers(v)
        fused = hasattr(self.k, "edges")
        if not (fused and chain and self._w_of is v):
            self.k.halo_w(self.U, v, w_send)
        self._w_of = None
        reqs = self.exchange(v, w_send, v_hi, w_lo)
        interior, edges = boundary_ranges(self.k.nt(v))
        if interior is not None:
            with _maybe(timer):
                self.k.sweep(self.U, v, out, interior, v_hi, w_lo)
        for r in reqs:
            r.wait()  # the sends have left w_send: the edges launch may overwrite it
        if fused:
            self.k.edges(self.U, v, out, v_hi, w_lo, w_send)
            self._w_of = out
        else:
            for rng in edges:
                self.k.sweep(self.U, v, out, rng, v_hi, w_lo)
        return out

    def launches_per_apply(self, chained: bool = False) -> int:
        """Kernel launches of one application (halo pack unless chained, interior, boundary slices)."""
        if self.world == 1:
            return 1
        interior, edges = boundary_ranges(self.k.nt(self.U))
        if hasattr(self.k, "edges"):
            return (0 if chained else 1) + (interior is not None) + 1
        return 1 + (interior is not None) + len(edges)

    def apply_n(self, v, scratch, applications: int):
        """v <- D v `applications` times (ping-pong); returns the buffer holding the result."""
        a, b = v, scratch
        for i in range(applications):
            self.apply(a, b, chain=i > 0)
            a, b = b, a
        return a
