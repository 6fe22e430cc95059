"""Thin ctypes binding of libtc (include/tc.h, include/tc_synth.h).

Argument marshalling only: torch tensors provide device / pinned memory (``data_ptr()``) and
torch streams provide ``cudaStream_t`` handles; every step of the codec runs in libtc's CUDA
kernels.  There is NO fallback: if libtc.so is missing or fails to load, importing this
module raises, and no function here ever computes a result on the host.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
# TC_LIB_PATH: an experiment build of the same sources (tools/, A/B runs); default the in-tree one
LIB_PATH = os.environ.get("TC_LIB_PATH") or os.path.join(PKG, "libtc.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

OK, ERR_INVALID, ERR_NOMEM, ERR_CUDA, ERR_NCCL = 0, 1, 2, 3, 4
ERR_CORRUPT, ERR_PROTOCOL, ERR_UNAVAILABLE, ERR_CAPACITY, ERR_INTERNAL = 5, 6, 7, 8, 9
D2H, H2D = 0, 1
TO_NEXT, TO_PREV = 0, 1
MAX_SEGMENTS, MAX_FOLD = 16, 64

u64, u32, vp, cint = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int


class Segment(ctypes.Structure):
    _fields_ = [("ref", vp), ("cur", vp), ("n_words", u64), ("word_bytes", u32), ("reserved", u32)]


class EncodeOpts(ctypes.Structure):
    _fields_ = [("tile_words", u32), ("advance_ref", u32), ("chunk_words", u64), ("index_mode", u32),
                ("reserved", u32)]


class GradOpts(ctypes.Structure):
    """tc_grad_opts (include/tc_grad.h)."""
    _fields_ = [("small_threshold", u64), ("k", ctypes.c_double), ("sample_size", u32), ("reserved", u32),
                ("chunk_elems", u64)]


class AdamHP(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double)]


class AdamState(ctypes.Structure):
    _fields_ = [("master", vp), ("m", vp), ("v", vp), ("w16", vp), ("n", u64)]


class TcError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {_status_string(status)} ({detail})")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libtc.so not found at {LIB_PATH}; build it with `python -m paper_2605_17821_b200.build` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(LIB_PATH)
    L.tc_status_string.restype = ctypes.c_char_p
    L.tc_status_string.argtypes = [cint]
    L.tc_last_error.restype = ctypes.c_char_p
    L.tc_last_error.argtypes = []
    L.tc_abi_version.restype = cint
    L.tc_ctx_create.argtypes = [cint, ctypes.POINTER(vp)]
    L.tc_ctx_destroy.argtypes = [vp]
    L.tc_ctx_check.argtypes = [vp, vp]
    L.tc_ctx_launches.restype = u64
    L.tc_ctx_launches.argtypes = [vp]
    L.tc_ctx_set_fold_dense_permille.argtypes = [vp, u32]
    L.tc_ctx_set_push_ctas.argtypes = [vp, u32]
    L.tc_ctx_set_fold_max_records.argtypes = [vp, u64]
    L.tc_diff_bound.argtypes = [ctypes.POINTER(Segment), cint, ctypes.POINTER(EncodeOpts),
                                ctypes.POINTER(u64)]
    L.tc_diff_encode.argtypes = [vp, ctypes.POINTER(Segment), cint, ctypes.POINTER(EncodeOpts), u64, u64,
                                 vp, u64, vp, vp]
    L.tc_stage_host.argtypes = [vp, vp, u64, cint, vp]
    L.tc_diff_bound_range.argtypes = [ctypes.POINTER(Segment), ctypes.POINTER(EncodeOpts), u64, u64,
                                      ctypes.POINTER(u64)]
    L.tc_diff_encode_range.argtypes = [vp, ctypes.POINTER(Segment), u32, ctypes.POINTER(EncodeOpts), u64, u64,
                                       u64, u64, vp, u64, vp, vp]
    L.tc_host_alloc.argtypes = [u64, ctypes.POINTER(vp)]
    L.tc_host_free.argtypes = [vp]
    L.tc_comm_get_unique_id.argtypes = [ctypes.c_char_p]
    L.tc_comm_init.argtypes = [cint, cint, cint, ctypes.c_char_p, ctypes.POINTER(vp)]
    L.tc_comm_destroy.argtypes = [vp]
    L.tc_replicate_peer.argtypes = [vp, vp, vp, vp, u64, ctypes.POINTER(u64), cint, vp]
    L.tc_diff_apply.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(u64), ctypes.POINTER(u32), cint, u64,
                                ctypes.POINTER(vp), ctypes.POINTER(u64), cint, vp]
    L.tc_synth_base.argtypes = [vp, u64, u32, u64, u32, u64, vp]
    L.tc_synth_step.argtypes = [vp, u64, u32, u64, u32, u64, u64, cint, u64, vp]
    L.tc_ipc_alloc.argtypes = [u64, ctypes.POINTER(vp), ctypes.c_char_p]
    L.tc_ipc_free.argtypes = [vp]
    L.tc_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.tc_ipc_close.argtypes = [vp]
    L.tc_push_peer.argtypes = [vp, vp, vp, vp, u64, vp, u64, vp]
    L.tc_diff_encode_push.argtypes = [vp, ctypes.POINTER(Segment), cint, ctypes.POINTER(EncodeOpts), u64, u64,
                                      vp, u64, vp, vp, u64, vp, vp]
    L.tc_peer_wait.argtypes = [vp, vp, u64, vp, vp]
    L.tc_grad_bound.argtypes = [u64, ctypes.POINTER(GradOpts), ctypes.POINTER(u64)]
    L.tc_grad_compress.argtypes = [vp, vp, u64, ctypes.POINTER(GradOpts), u64, vp, u64, vp, vp]
    L.tc_grad_decompress.argtypes = [vp, vp, u64, vp, u64, vp]
    L.tc_adam_step.argtypes = [vp, ctypes.POINTER(AdamState), vp, ctypes.POINTER(AdamHP), u64, vp]
    L.tc_adam_replay.argtypes = [vp, ctypes.POINTER(AdamState), ctypes.POINTER(vp), ctypes.POINTER(u64), cint,
                                 ctypes.POINTER(AdamHP), u64, vp, vp]
    L.tc_adam_step_encode.argtypes = [vp, ctypes.POINTER(AdamState), vp, ctypes.POINTER(AdamHP), u64,
                                      ctypes.POINTER(EncodeOpts), vp, u64, vp, vp]
    for name in ("tc_grad_bound", "tc_grad_compress", "tc_grad_decompress", "tc_adam_step", "tc_adam_replay",
                 "tc_adam_step_encode"):
        getattr(L, name).restype = cint
    for name in ("tc_ipc_alloc", "tc_ipc_free", "tc_ipc_open", "tc_ipc_close", "tc_push_peer",
                 "tc_diff_encode_push", "tc_peer_wait"):
        getattr(L, name).restype = cint
    for name in ("tc_ctx_create", "tc_ctx_destroy", "tc_ctx_check", "tc_diff_bound", "tc_diff_encode",
                 "tc_stage_host", "tc_diff_bound_range", "tc_diff_encode_range", "tc_host_alloc", "tc_host_free", "tc_comm_get_unique_id", "tc_comm_init", "tc_comm_destroy",
                 "tc_replicate_peer", "tc_diff_apply", "tc_synth_base", "tc_synth_step"):
        getattr(L, name).restype = cint
    return L


LIB = _load()


def _status_string(s: int) -> str:
    return LIB.tc_status_string(s).decode()


def _check(rc: int, where: str):
    if rc != OK:
        raise TcError(rc, where, LIB.tc_last_error().decode())


def header_symbols():
    """Every function the public headers declare (for the ABI export test)."""
    names = []
    for h in ("tc.h", "tc_synth.h", "tc_grad.h"):
        with open(os.path.join(INCLUDE, h)) as fh:
            txt = fh.read()
        names += re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tc_\w+)\s*\(", txt, re.M)
    return sorted(set(names))


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


FORMAT_MASK, FORMAT_INDEX, FORMAT_FULL = 0, 1, 2  # tc_encode_opts.index_mode (include/tc.h)


def _opts(tile_words=4096, chunk_words=1 << 28, advance_ref=True, index_mode=False, full=False) -> EncodeOpts:
    fmt = FORMAT_FULL if full else (FORMAT_INDEX if index_mode else FORMAT_MASK)
    return EncodeOpts(tile_words, 1 if advance_ref else 0, chunk_words, fmt, 0)


def _wb(t: torch.Tensor) -> int:
    wb = t.element_size()
    if wb not in (2, 4):
        raise TcError(ERR_INVALID, "segment", f"element size {wb} not in (2, 4)")
    return wb


def segments(ref, cur):
    if len(ref) != len(cur):
        raise TcError(ERR_INVALID, "segments", "ref/cur length mismatch")
    arr = (Segment * len(ref))()
    for i, (r, c) in enumerate(zip(ref, cur)):
        if r.numel() != c.numel() or r.element_size() != c.element_size():
            raise TcError(ERR_INVALID, "segments", f"segment {i} shape mismatch")
        arr[i] = Segment(r.data_ptr() if r.numel() else None, c.data_ptr() if c.numel() else None,
                         r.numel(), _wb(r), 0)
    return arr


def layout_segments(sizes, word_bytes):
    arr = (Segment * len(sizes))()
    for i, (n, w) in enumerate(zip(sizes, word_bytes)):
        arr[i] = Segment(None, None, int(n), int(w), 0)
    return arr


def diff_bound(sizes, word_bytes, tile_words=4096, chunk_words=1 << 28, index_mode=False, full=False) -> int:
    segs = layout_segments(sizes, word_bytes)
    o = _opts(tile_words, chunk_words, True, index_mode, full)
    out = u64(0)
    _check(LIB.tc_diff_bound(segs, len(sizes), ctypes.byref(o), ctypes.byref(out)), "tc_diff_bound")
    return out.value


class Ctx:
    """tc_ctx: per-device scratch + sticky device error."""

    def __init__(self, device: int | None = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        h = vp()
        _check(LIB.tc_ctx_create(device, ctypes.byref(h)), "tc_ctx_create")
        self.h = h

    def check(self, stream=None):
        _check(LIB.tc_ctx_check(self.h, _stream(stream)), "tc_ctx_check")

    def check_status(self, stream=None) -> int:
        return LIB.tc_ctx_check(self.h, _stream(stream))

    @property
    def launches(self) -> int:
        return int(LIB.tc_ctx_launches(self.h))

    def set_push_ctas(self, ctas: int):
        """CTAs of tc_push_peer on this ctx (include/tc.h); 0 = default."""
        _check(LIB.tc_ctx_set_push_ctas(self.h, int(ctas)), "tc_ctx_set_push_ctas")

    def set_fold_max_records(self, records: int):
        """tc_ctx_set_fold_max_records: records per diff the later folds hold at most (0 = no bound)."""
        _check(LIB.tc_ctx_set_fold_max_records(self.h, int(records)), "tc_ctx_set_fold_max_records")

    def set_fold_dense_permille(self, permille: int):
        """Restore strategy threshold (include/tc.h): 0 = always stream, 2**32-1 = always scatter."""
        _check(LIB.tc_ctx_set_fold_dense_permille(self.h, int(permille)), "tc_ctx_set_fold_dense_permille")

    def close(self):
        if self.h:
            LIB.tc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def diff_encode(ctx: Ctx, ref, cur, out: torch.Tensor, out_bytes: torch.Tensor, version: int, ref_version: int,
                tile_words=4096, chunk_words=1 << 28, advance_ref=True, stream=None, index_mode=False, full=False):
    """Enqueue tc_diff_encode.  ``out`` uint8 CUDA tensor, ``out_bytes`` int64 CUDA tensor [1].
    Record format: mask (default), index (``index_mode``) or full (``full``: every word)."""
    segs = segments(ref, cur)
    o = _opts(tile_words, chunk_words, advance_ref, index_mode, full)
    _check(LIB.tc_diff_encode(ctx.h, segs, len(ref), ctypes.byref(o), version, ref_version, out.data_ptr(),
                              out.numel() * out.element_size(), out_bytes.data_ptr(), _stream(stream)),
           "tc_diff_encode")


IPC_HANDLE_BYTES = 64


class IpcBuffer:
    """Receiver side of the NVLink push (tc_ipc_alloc): device memory in this GPU whose IPC
    handle (``.handle``, 64 bytes) the ring neighbour maps.  ``.tensor`` is a zero-copy uint8
    CUDA view (``__cuda_array_interface__``)."""

    def __init__(self, nbytes: int):
        p = vp()
        h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(LIB.tc_ipc_alloc(int(nbytes), ctypes.byref(p), h), "tc_ipc_alloc")
        self.ptr, self.nbytes, self.handle = p.value, int(nbytes), h.raw
        self.__cuda_array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                         "version": 2, "strides": None}
        self.tensor = torch.as_tensor(self, device="cuda")

    def data_ptr(self):
        return self.ptr

    def numel(self):
        return self.nbytes

    def element_size(self):
        return 1

    def free(self):
        if self.ptr:
            self.tensor = None
            LIB.tc_ipc_free(self.ptr)
            self.ptr = None


class PeerMapping:
    """Sender side: a neighbour's IpcBuffer mapped into this process (tc_ipc_open)."""

    def __init__(self, handle: bytes, nbytes: int):
        p = vp()
        _check(LIB.tc_ipc_open(handle, ctypes.byref(p)), "tc_ipc_open")
        self.ptr, self.nbytes = p.value, int(nbytes)

    def data_ptr(self):
        return self.ptr

    def close(self):
        if self.ptr:
            LIB.tc_ipc_close(self.ptr)
            self.ptr = None


def push_peer(ctx: Ctx, src: torch.Tensor, src_bytes, peer_dst, peer_cap: int, peer_mailbox, version: int,
              stream=None):
    """Enqueue tc_push_peer: the record at ``src`` (length: the u64 at ``src_bytes``) -> the peer slot."""
    _check(LIB.tc_push_peer(ctx.h, src.data_ptr(), src_bytes.data_ptr(), peer_dst.data_ptr(), int(peer_cap),
                            peer_mailbox.data_ptr(), version, _stream(stream)), "tc_push_peer")


def diff_encode_push(ctx: Ctx, ref, cur, out: torch.Tensor, out_bytes, version: int, ref_version: int, peer_dst,
                     peer_cap: int, peer_mailbox, tile_words=4096, chunk_words=1 << 28, advance_ref=True,
                     stream=None, index_mode=False, full=False):
    """Enqueue tc_diff_encode_push: the encoder writes the record into `out` AND the ring
    neighbour's slot (fused Tier-2 emit) and publishes its mailbox."""
    segs = segments(ref, cur)
    o = _opts(tile_words, chunk_words, advance_ref, index_mode, full)
    _check(LIB.tc_diff_encode_push(ctx.h, segs, len(ref), ctypes.byref(o), version, ref_version, out.data_ptr(),
                                   out.numel() * out.element_size(), out_bytes.data_ptr(), peer_dst.data_ptr(),
                                   int(peer_cap), peer_mailbox.data_ptr(), _stream(stream)), "tc_diff_encode_push")


def peer_wait(ctx: Ctx, mailbox, version: int, bytes_out=None, stream=None):
    """Enqueue tc_peer_wait on this GPU's mailbox (IpcBuffer) for ``version``."""
    _check(LIB.tc_peer_wait(ctx.h, mailbox.data_ptr(), version, None if bytes_out is None else bytes_out.data_ptr(),
                            _stream(stream)), "tc_peer_wait")


def diff_bound_range(n_words: int, word_bytes: int, first_chunk: int, n_chunks: int, tile_words=4096,
                     chunk_words=1 << 28, index_mode=False, full=False) -> int:
    seg = Segment(None, None, int(n_words), int(word_bytes), 0)
    o = _opts(tile_words, chunk_words, True, index_mode, full)
    out = u64(0)
    _check(LIB.tc_diff_bound_range(ctypes.byref(seg), ctypes.byref(o), first_chunk, n_chunks, ctypes.byref(out)),
           "tc_diff_bound_range")
    return out.value


def diff_encode_range(ctx: Ctx, ref: torch.Tensor, cur: torch.Tensor, segment_id: int, first_chunk: int,
                      n_chunks: int, out: torch.Tensor, out_bytes: torch.Tensor, version: int, ref_version: int,
                      tile_words=4096, chunk_words=1 << 28, advance_ref=True, stream=None, index_mode=False,
                      full=False):
    """Enqueue tc_diff_encode_range (the records of chunks [first_chunk, first_chunk+n_chunks) of
    one segment, byte-identical to that part of the full encode)."""
    seg = segments([ref], [cur])
    o = _opts(tile_words, chunk_words, advance_ref, index_mode, full)
    _check(LIB.tc_diff_encode_range(ctx.h, seg, segment_id, ctypes.byref(o), first_chunk, n_chunks, version,
                                    ref_version, out.data_ptr(), out.numel() * out.element_size(),
                                    out_bytes.data_ptr(), _stream(stream)), "tc_diff_encode_range")


def diff_apply(ctx: Ctx, state, state_version: int, records, record_bytes, stream=None):
    """Enqueue tc_diff_apply: fold ``records`` (oldest first) onto ``state`` in place."""
    n = len(state)
    sp = (vp * n)(*[s.data_ptr() if s.numel() else None for s in state])
    nw = (u64 * n)(*[s.numel() for s in state])
    wb = (u32 * n)(*[_wb(s) for s in state])
    k = len(records)
    rp = (vp * k)(*[r.data_ptr() for r in records])
    rb = (u64 * k)(*[int(b) for b in record_bytes])
    _check(LIB.tc_diff_apply(ctx.h, sp, nw, wb, n, state_version, rp, rb, k, _stream(stream)), "tc_diff_apply")


def stage_host(dst: torch.Tensor, src: torch.Tensor, nbytes: int, direction: int, stream=None):
    _check(LIB.tc_stage_host(dst.data_ptr(), src.data_ptr(), int(nbytes), direction, _stream(stream)),
           "tc_stage_host")


class HostBuffer:
    """A page-locked host buffer from tc_host_alloc (the Tier-1 ring slot), viewed as a CPU uint8
    tensor.  Freed with tc_host_free when this object is collected."""

    def __init__(self, nbytes: int):
        p = vp()
        _check(LIB.tc_host_alloc(int(nbytes), ctypes.byref(p)), "tc_host_alloc")
        self.ptr = p.value
        self.nbytes = int(nbytes)
        if nbytes:
            arr = (ctypes.c_uint8 * self.nbytes).from_address(self.ptr)
            self.tensor = torch.frombuffer(arr, dtype=torch.uint8)
        else:
            self.tensor = torch.empty(0, dtype=torch.uint8)

    def view(self, dtype, n=None):
        t = self.tensor.view(dtype)
        return t if n is None else t[:n]

    def data_ptr(self):
        return self.ptr

    def numel(self):
        return self.nbytes

    def element_size(self):
        return 1

    def numpy(self):
        return self.tensor.numpy()

    def free(self):
        if self.ptr:
            self.tensor = None
            LIB.tc_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Comm:
    """tc_comm: libtc's own NCCL communicator for the Tier-2 ring ("isolated
    communication groups").  The unique id is broadcast over a torch.distributed group."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist

        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(LIB.tc_comm_get_unique_id(buf), "tc_comm_get_unique_id")
        if world > 1:
            t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone()
            if dist.get_backend(group) == "nccl":
                t = t.cuda(device)
            dist.broadcast(t, src=0, group=group)
            buf = ctypes.create_string_buffer(bytes(t.cpu().tolist()), 128)
        h = vp()
        _check(LIB.tc_comm_init(world, rank, device, buf, ctypes.byref(h)), "tc_comm_init")
        self.h = h
        self.rank, self.world = rank, world

    def replicate_peer(self, send: torch.Tensor, send_bytes: torch.Tensor, recv: torch.Tensor,
                       direction: int = TO_NEXT, stream=None) -> int:
        got = u64(0)
        _check(LIB.tc_replicate_peer(self.h, send.data_ptr(), send_bytes.data_ptr(), recv.data_ptr(),
                                     recv.numel() * recv.element_size(), ctypes.byref(got), direction,
                                     _stream(stream)), "tc_replicate_peer")
        return got.value

    def close(self):
        if self.h:
            LIB.tc_comm_destroy(self.h)
            self.h = None


def synth_base(dst: torch.Tensor, seed: int, seg: int, start: int = 0, stream=None):
    _check(LIB.tc_synth_base(dst.data_ptr(), dst.numel(), _wb(dst), seed, seg, start, _stream(stream)),
           "tc_synth_base")


def synth_step(words: torch.Tensor, seed: int, seg: int, t: int, p53: int, structure: int = 0, start: int = 0,
               stream=None):
    _check(LIB.tc_synth_step(words.data_ptr(), words.numel(), _wb(words), seed, seg, t, p53, structure, start,
                             _stream(stream)), "tc_synth_step")


# ------------------------------------------------ the paper's lossy differential (tc_grad.h)
def _gopts(k=0.01, small_threshold=100_000, sample_size=4096, chunk_elems=(1 << 31) - 4096):
    return GradOpts(int(small_threshold), float(k), int(sample_size), 0, int(chunk_elems))


def grad_bound(n: int, **opts) -> int:
    out = u64(0)
    o = _gopts(**opts)
    _check(LIB.tc_grad_bound(int(n), ctypes.byref(o), ctypes.byref(out)), "tc_grad_bound")
    return out.value


def grad_compress(ctx: Ctx, grad: torch.Tensor, seed: int, out: torch.Tensor, out_bytes: torch.Tensor,
                  stream=None, **opts):
    """Enqueue tc_grad_compress of the fp32 CUDA tensor ``grad`` into ``out`` (uint8)."""
    o = _gopts(**opts)
    _check(LIB.tc_grad_compress(ctx.h, grad.data_ptr(), grad.numel(), ctypes.byref(o), int(seed), out.data_ptr(),
                                out.numel() * out.element_size(), out_bytes.data_ptr(), _stream(stream)),
           "tc_grad_compress")


def grad_decompress(ctx: Ctx, payload: torch.Tensor, nbytes: int, out: torch.Tensor, stream=None):
    _check(LIB.tc_grad_decompress(ctx.h, payload.data_ptr(), int(nbytes), out.data_ptr(), out.numel(),
                                  _stream(stream)), "tc_grad_decompress")


def _adam(master, m, v, w16):
    return AdamState(master.data_ptr(), m.data_ptr(), v.data_ptr(), w16.data_ptr(), master.numel())


def _hp(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    return AdamHP(lr, beta1, beta2, eps)


def adam_step(ctx: Ctx, master, m, v, w16, grad, step: int, stream=None, **hp):
    """Enqueue tc_adam_step (fp32 master/m/v, int16 tensor of bf16 bits w16, fp32 grad; 1-based step)."""
    st, h = _adam(master, m, v, w16), _hp(**hp)
    _check(LIB.tc_adam_step(ctx.h, ctypes.byref(st), grad.data_ptr(), ctypes.byref(h), int(step), _stream(stream)),
           "tc_adam_step")


def adam_replay(ctx: Ctx, master, m, v, w16, payloads, payload_bytes, first_step: int, scratch, stream=None, **hp):
    """Enqueue tc_adam_replay: payloads[:-1] fused, the last through the native step."""
    st, h = _adam(master, m, v, w16), _hp(**hp)
    k = len(payloads)
    pp = (vp * k)(*[p.data_ptr() for p in payloads])
    pb = (u64 * k)(*[int(b) for b in payload_bytes])
    _check(LIB.tc_adam_replay(ctx.h, ctypes.byref(st), pp, pb, k, ctypes.byref(h), int(first_step),
                              scratch.data_ptr(), _stream(stream)), "tc_adam_replay")


def adam_step_encode(ctx: Ctx, master, m, v, w16, grad, step: int, out: torch.Tensor, out_bytes, tile_words=4096,
                     chunk_words=1 << 28, index_mode=False, stream=None, full=False, **hp):
    """Enqueue tc_adam_step_encode: the Adam step + the lossless diff of its update (segments w16,
    master, m, v) into ``out``; ``full`` = full records written in the Adam pass itself."""
    st, h = _adam(master, m, v, w16), _hp(**hp)
    o = _opts(tile_words, chunk_words, False, index_mode, full)
    _check(LIB.tc_adam_step_encode(ctx.h, ctypes.byref(st), grad.data_ptr(), ctypes.byref(h), int(step), ctypes.byref(o),
                                   out.data_ptr(), out.numel() * out.element_size(), out_bytes.data_ptr(),
                                   _stream(stream)), "tc_adam_step_encode")
