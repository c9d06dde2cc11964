"""Fused compute + NVLink halo push for the t-slab NN sweep (csrc/p2p.cu).

``slab.SlabSweep`` exchanges the two halo faces with NCCL send/recv around the
boundary compute.  ``P2PSlabSweep`` removes the collective: the kernel that
computes a rank's two boundary slices stores the next application's halos
directly into its neighbours' windows (device memory mapped into this process
with CUDA IPC) and releases a system-scope flag; the neighbours' boundary
kernels wait on that flag.  Per application on every rank:

    k_p2p_boundary (wait flags >= e+1; t = 0, nt-1; push halos of e+1; release e+2)
    interior slices [1, nt-1)                 -- overlaps the peers' pushes

One process per GPU; the windows' IPC handles are exchanged once over
torch.distributed.  With one rank the window is its own peer (the protocol runs
unchanged on a single GPU).  Results are bit-identical to the periodic sweep.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .lattice import Field

_SFX = {torch.float32: "f32", torch.float64: "f64"}


class P2PSlabSweep:
    """Slab NN sweep whose boundary kernel pushes the halos to the neighbours over NVLink."""

    def __init__(self, U: Field, group=None, mode: str = "exact"):
        import torch.distributed as dist

        from .sweeps import _mode

        if U.kind != "mat4":
            raise ValueError("P2PSlabSweep needs U of kind 'mat4'")
        self.U = U
        self.mode = _mode(mode)
        self.dist = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.dist else 0
        self.world = dist.get_world_size(group) if self.dist else 1
        self.group = group
        lat = U.lattice
        esz = torch.tensor([], dtype=U.dtype).element_size()
        nbytes = int(_lib.load().su3g_p2p_window_bytes(lat.nx, lat.ny, lat.nz, esz))
        if nbytes <= 0:
            raise ValueError("invalid lattice for the P2P window")
        self.window = torch.zeros(nbytes, dtype=torch.uint8, device=U.device)
        self.ctrl_offset = int(_lib.load().su3g_p2p_ctrl_offset(lat.nx, lat.ny, lat.nz, esz))
        self._opened = []
        lo, hi = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        if self.world == 1:
            self.win_lo = self.win_hi = self.window.data_ptr()
        else:
            handle = ctypes.create_string_buffer(_lib.SU3G_IPC_HANDLE_BYTES)
            _lib.call("su3g_ipc_get_handle", ctypes.c_void_p(self.window.data_ptr()), handle)
            handles = [None] * self.world
            dist.all_gather_object(handles, handle.raw, group=group)
            ptrs = {}
            for peer in {lo, hi}:
                if peer == self.rank:
                    ptrs[peer] = self.window.data_ptr()
                    continue
                p = ctypes.c_void_p()
                buf = ctypes.create_string_buffer(bytes(handles[peer]), _lib.SU3G_IPC_HANDLE_BYTES)
                _lib.call("su3g_ipc_open_handle", buf, ctypes.byref(p))
                self._opened.append(p)
                ptrs[peer] = p.value
            self.win_lo, self.win_hi = ptrs[lo], ptrs[hi]
        self.epoch = 0
        self._primed_for = None  # data_ptr of the field whose halos are in flight for self.epoch

    def _barrier(self):
        torch.cuda.synchronize(self.U.device)
        if self.dist and self.world > 1:
            import torch.distributed as dist

            dist.barrier(group=self.group)

    def _needs_prime(self, v: Field) -> bool:
        """Whether v is a fresh source -- decided collectively: if any rank must prime, every rank
        primes (a per-rank pointer test could diverge when the allocator hands one rank a fresh v at
        the address of its previous out, and the epochs would then drift apart)."""
        need = self._primed_for != v.data.data_ptr()
        if self.dist and self.world > 1:
            import torch.distributed as dist

            flag = torch.tensor([int(need)], dtype=torch.int32, device=self.U.device)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
            need = bool(flag.item())
        return need

    def invalidate(self) -> None:
        """Forget the in-flight halos: call after writing a source field in place."""
        self._primed_for = None

    def apply(self, v: Field, out: Field, chain: bool | None = None) -> Field:
        """out = D v for this rank's slab (collective: every rank calls it in the same order).

        Consecutive calls that feed one call's ``out`` back as the next ``v`` need no
        priming: the boundary kernel already pushed those halos.  Any other source is
        primed first (host barrier + su3g_p2p_prime); if ``out`` was modified in place
        before being fed back, call ``invalidate()`` first.

        ``chain`` makes the decision explicit and identical on every rank: True = v is the
        previous call's out (raises if it is not), False = prime.  None decides collectively
        (an all-reduce over the ranks, one host round trip per call).
        """
        if v.kind != "vec" or out.kind != "vec" or v.lattice != self.U.lattice or v.dtype != self.U.dtype:
            raise ValueError("v and out must be 'vec' fields on U's slab lattice and dtype")
        lat = self.U.lattice
        sfx = _SFX[self.U.dtype]
        stream = torch.cuda.current_stream(self.U.device).cuda_stream
        me = ctypes.c_void_p(self.window.data_ptr())
        lo, hi = ctypes.c_void_p(self.win_lo), ctypes.c_void_p(self.win_hi)
        if chain is None:
            prime = self._needs_prime(v)
        elif chain:
            if self._primed_for != v.data.data_ptr():
                raise ValueError("chain=True, but v is not the previous application's out (or was invalidated)")
            prime = False
        else:
            prime = True
        if prime:
            # fresh source: all ranks' earlier launches must be done before the windows are rewritten,
            # and the epoch skips ahead so no stale flag can satisfy the next wait
            self._barrier()
            self.epoch += 1
            _lib.call(f"su3g_p2p_prime_{sfx}", self.U.data.data_ptr(), v.data.data_ptr(), lat.nx, lat.ny, lat.nz,
                      lat.nt, me, lo, hi, self.epoch, self.mode, stream)
        _lib.call(f"su3g_p2p_nn_sweep_{sfx}", self.U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
                  lat.nx, lat.ny, lat.nz, lat.nt, me, lo, hi, self.epoch, self.mode, stream)
        self.epoch += 1
        self._primed_for = out.data.data_ptr()  # the boundary kernel pushed out's halos for the next epoch
        return out

    def apply_n(self, v: Field, applications: int, scratch: Field | None = None) -> Field:
        """v <- D v `applications` times (ping-pong); the initial v is always primed as a fresh source."""
        self.invalidate()
        a, b = v, (scratch if scratch is not None else v.empty_like())
        for i in range(applications):
            self.apply(a, b, chain=i > 0)
            a, b = b, a
        self.check()
        return a

    def check(self) -> None:
        """Raise if a halo wait timed out (the boundary kernel's bounded spin set the error word)."""
        if self.error():
            raise RuntimeError("P2P halo exchange: a flag wait timed out (protocol failure); results are invalid")

    def error(self) -> int:
        """The window's error word: 1 if a halo wait timed out (protocol failure), else 0."""
        return int(self.window[self.ctrl_offset + 20: self.ctrl_offset + 24].view(torch.int32).item())

    def close(self):
        torch.cuda.synchronize(self.U.device)
        for p in self._opened:
            _lib.call("su3g_ipc_close", p)
        self._opened = []
