"""Native (C ABI) t-slab NN sweep: NCCL communicator handles of libsu3g.

``slab.SlabSweep`` drives the slab decomposition from Python over
torch.distributed; this module binds the same schedule implemented in C++
(csrc/comm.cu) for hosts that talk to the C ABI directly:

    uid = NativeComm.unique_id()                     # on one rank, then broadcast the 128 bytes
    comm = NativeComm(world, rank, uid)              # collective; the rank's GPU current
    out = native_slab_sweep(comm, U, v, out)         # one application of D on this rank's slab
    comm.close()

A one-rank communicator exchanges with itself, so the full exchange schedule
(pack, grouped send/recv on the comm stream, interior overlap, boundary) runs
and is checked on a single GPU.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .lattice import Field

_SFX = {torch.float32: "f32", torch.float64: "f64"}


class NativeComm:
    """An su3g_comm_t: an NCCL communicator plus the comm stream, events and halo buffers."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        if len(unique_id) != _lib.SU3G_COMM_ID_BYTES:
            raise ValueError(f"unique_id must be {_lib.SU3G_COMM_ID_BYTES} bytes")
        self._h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(unique_id), _lib.SU3G_COMM_ID_BYTES)
        _lib.call("su3g_comm_init", int(nranks), int(rank), buf, ctypes.byref(self._h))
        self.nranks, self.rank = int(nranks), int(rank)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(_lib.SU3G_COMM_ID_BYTES)
        _lib.call("su3g_comm_unique_id", buf)
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "NativeComm":
        """Build over an initialised torch.distributed group (rank 0's id broadcast as a tensor)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        uid = torch.zeros(_lib.SU3G_COMM_ID_BYTES, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(cls.unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0, group=group)
        return cls(world, rank, bytes(uid.cpu().numpy().tobytes()))

    @property
    def handle(self):
        if self._h is None or not self._h.value:
            raise ValueError("communicator is closed")
        return self._h

    def check(self, timeout_s: float | None = 60.0) -> None:
        """Wait for the last halo exchange, watching NCCL's asynchronous error state (su3g_comm_check).
        A failed or stalled exchange (dead peer) aborts the communicator and raises RuntimeError."""
        ms = -1 if timeout_s is None else int(timeout_s * 1000)
        _lib.call("su3g_comm_check", self.handle, ms)  # the handle stays valid for close()

    def close(self) -> None:
        if self._h is not None and self._h.value:
            h, self._h = self._h, None
            _lib.call("su3g_comm_destroy", h)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def native_slab_sweep(comm: NativeComm, U: Field, v: Field, out: Field | None = None, mode: str = "exact") -> Field:
    """out = D v on this rank's t-slab, halos exchanged by libsu3g over NCCL (su3g_slab_nn_sweep)."""
    from .sweeps import _mode

    if U.kind != "mat4" or v.kind != "vec" or U.lattice != v.lattice or U.dtype != v.dtype:
        raise ValueError("native_slab_sweep needs U ('mat4') and v ('vec') on the same slab lattice and dtype")
    if out is None:
        out = v.empty_like()
    lat = U.lattice
    _lib.call(
        f"su3g_slab_nn_sweep_{_SFX[U.dtype]}", comm.handle, U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
        lat.nx, lat.ny, lat.nz, lat.nt, _mode(mode), torch.cuda.current_stream(U.device).cuda_stream,
    )
    return out


def native_slab_apply(comm: NativeComm, U: Field, v: Field, applications: int, scratch: Field | None = None,
                      mode: str = "exact") -> Field:
    """v <- D v, `applications` times across the ranks, ping-ponging two buffers; returns the final field."""
    a, b = v, (scratch if scratch is not None else v.empty_like())
    for _ in range(applications):
        native_slab_sweep(comm, U, a, b, mode)
        a, b = b, a
    comm.check()
    return a
