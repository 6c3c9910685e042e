"""Python face of the C ABI: ``Plan`` and the host-only queries.

PyTorch provides device memory and streams; every step of the transform runs
in libffst.so's kernels (include/ffst.h).  Names follow the paper's API
(shearletTransformSpect / inverseShearletTransformSpect) and
the boundary of SURVEY.md 8(b).
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import PlanDesc, check, lib

KIND_NAMES = {0: "lowpass", 1: "h", 2: "v", 3: "x"}
_DTYPES = {torch.float32: 0, torch.float64: 1}
_CDTYPES = {torch.float32: torch.complex64, torch.float64: torch.complex128}
_VARIANTS = {"classic": 0, "smooth": 1, "user": 2}
_POLICIES = {"lpt": 0, "round_robin": 1}


def scales_for_size(n: int) -> int:
    """j0 = floor(1/2 log2 n)."""
    j0 = C.c_int()
    check(lib.ffst_scales_for_size(int(n), C.byref(j0)), "ffst_scales_for_size")
    return j0.value


def num_shearlets(j0: int) -> int:
    """eta = 2^(j0+2) - 3."""
    return lib.ffst_num_shearlets(int(j0))


def index_to_params(j0: int, index: int):
    """0-based flat index -> (kind, j, k) (Sec. 3.5.1)."""
    kind, j, k = C.c_int(), C.c_int(), C.c_int()
    check(lib.ffst_index_to_params(int(j0), int(index), C.byref(kind), C.byref(j), C.byref(k)),
          "ffst_index_to_params")
    return kind.value, j.value, k.value


def params_to_index(j0: int, kind: int, j: int, k: int) -> int:
    i = C.c_int()
    check(lib.ffst_params_to_index(int(j0), int(kind), int(j), int(k), C.byref(i)), "ffst_params_to_index")
    return i.value


def plane_support(n: int, index: int, j0: int = 0):
    lo, hi = C.c_int(), C.c_int()
    check(lib.ffst_plane_support(int(n), int(j0), int(index), C.byref(lo), C.byref(hi)), "ffst_plane_support")
    return lo.value, hi.value


def shard_planes(n: int, shard_count: int, shard_rank: int, policy: str = "lpt", j0: int = 0):
    """Global 0-based indices of the planes rank `shard_rank` owns (host-only)."""
    cnt = C.c_int()
    check(lib.ffst_shard_planes(int(n), int(j0), int(shard_count), int(shard_rank), _POLICIES[policy],
                                C.byref(cnt), None), "ffst_shard_planes")
    idx = (C.c_int * max(1, cnt.value))()
    check(lib.ffst_shard_planes(int(n), int(j0), int(shard_count), int(shard_rank), _POLICIES[policy],
                                C.byref(cnt), idx), "ffst_shard_planes")
    return [idx[i] for i in range(cnt.value)]


class NcclComm:
    """An NCCL communicator owned by the library's side of the boundary (ffst_nccl_comm_create):
    rank 0 creates the unique id, the ranks exchange it out of band (torch.distributed), every rank
    joins.  Passed to Plan(nccl_comm=...) so that the library runs the exchange steps itself."""

    def __init__(self, nranks: int, rank: int, device: int, unique_id: bytes):
        from ._lib import NcclId
        nid = NcclId()
        C.memmove(C.addressof(nid), unique_id, 128)
        h = C.c_void_p()
        check(lib.ffst_nccl_comm_create(C.byref(h), int(nranks), int(rank), C.byref(nid), int(device)),
              "ffst_nccl_comm_create")
        self.handle, self.nranks, self.rank = h, int(nranks), int(rank)

    @staticmethod
    def unique_id() -> bytes:
        from ._lib import NcclId
        nid = NcclId()
        check(lib.ffst_nccl_unique_id(C.byref(nid)), "ffst_nccl_unique_id")
        return C.string_at(C.addressof(nid), 128)

    def close(self):
        if getattr(self, "handle", None):
            lib.ffst_nccl_comm_destroy(self.handle)
            self.handle = None


def plane_is_nyquist(n: int, index: int, j0: int = 0) -> bool:
    v = C.c_int()
    check(lib.ffst_plane_is_nyquist(int(n), int(j0), int(index), C.byref(v)), "ffst_plane_is_nyquist")
    return bool(v.value)


def _check_buf(t, shape, dtype, device, what):
    """Caller buffers reach the C ABI only with the exact shape, dtype, device and layout the
    call reads or writes (the library trusts the sizes it is given)."""
    if not torch.is_tensor(t):
        raise ValueError(f"{what}: a torch tensor is required")
    dev_ok = (t.device.type == "cpu") if device == "cpu" else (t.device == device)
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not dev_ok or not t.is_contiguous():
        where = "host memory" if device == "cpu" else str(device)
        raise ValueError(f"{what}: expected a contiguous {dtype} tensor of shape {tuple(shape)} in {where}, "
                         f"got {t.dtype} {tuple(t.shape)} on {t.device}"
                         f"{'' if t.is_contiguous() else ' (not contiguous)'}")
    return t


def _stream_handle(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return C.c_void_p(stream.cuda_stream)


class Plan:
    """A forward/inverse FFST plan for n x n images on one CUDA device.

    ``shard_rank``/``shard_count`` select the planes of ``shard_planes`` (eta-sharding, DESIGN.md
    "Multi-GPU"; ``shard_policy`` "lpt" or "round_robin").  With ``nccl_comm`` (a ``NcclComm`` of
    the shard_count ranks) the library broadcasts the images from rank 0 in ``forward`` and sums
    the ranks' partial adjoints onto ``root`` in ``inverse``."""

    def __init__(self, n: int, batch: int = 1, dtype=torch.float32, device=None, j0: int = 0,
                 shard_rank: int = 0, shard_count: int = 1, variant: str = "classic",
                 spectra=None, centred: bool = True, shard_policy: str = "lpt", nccl_comm=None):
        if not torch.cuda.is_available():
            raise RuntimeError("FFST Plan needs a CUDA device (no CPU fallback)")
        if dtype not in _DTYPES:
            raise TypeError("dtype must be torch.float32 or torch.float64")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.dtype = dtype
        self.cdtype = _CDTYPES[dtype]
        if spectra is not None:
            variant = "user"
        elif variant not in _VARIANTS or variant == "user":
            raise ValueError("variant must be 'classic' (meyerShearletSpect) or 'smooth' (meyerNewShearletSpect)")
        self.variant = variant
        if shard_policy not in _POLICIES:
            raise ValueError("shard_policy must be 'lpt' or 'round_robin'")
        self.comm = nccl_comm
        desc = PlanDesc(int(n), int(j0), int(batch), _DTYPES[dtype], _VARIANTS[variant], self.device.index,
                        int(shard_rank), int(shard_count), _POLICIES[shard_policy],
                        nccl_comm.handle if nccl_comm is not None else None)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            torch.cuda.init()
            if spectra is None:
                check(lib.ffst_plan_create(C.byref(handle), C.byref(desc)), "ffst_plan_create")
            else:
                # user-supplied spectra: eta real n x n planes, copied by the plan
                if (not torch.is_tensor(spectra) or spectra.dtype != dtype or spectra.device != self.device
                        or spectra.dim() != 3 or tuple(spectra.shape[1:]) != (n, n)):
                    raise ValueError(f"spectra must be a {dtype} tensor (eta, {n}, {n}) on {self.device}")
                spectra = spectra.contiguous()
                torch.cuda.current_stream(self.device).synchronize()
                check(lib.ffst_plan_create_user(C.byref(handle), C.byref(desc), int(spectra.shape[0]),
                                                C.c_void_p(spectra.data_ptr()), int(bool(centred))),
                      "ffst_plan_create_user")
        self._h = handle
        vals = [C.c_int() for _ in range(5)]
        check(lib.ffst_plan_info(self._h, *[C.byref(v) for v in vals]), "ffst_plan_info")
        self.n, self.j0, self.eta, self.eta_local, self.batch = (v.value for v in vals)
        idx = (C.c_int * self.eta_local)()
        cnt = C.c_int()
        check(lib.ffst_plan_local_planes(self._h, C.byref(cnt), idx), "ffst_plan_local_planes")
        self.local_planes = list(idx)
        pth = C.c_int()
        check(lib.ffst_plan_path(self._h, C.byref(pth)), "ffst_plan_path")
        self.path = {0: "persistent", 1: "fused_small", 2: "arbitrary_n"}[pth.value]
        self.shard_rank, self.shard_count = int(shard_rank), int(shard_count)
        self._reserved = {self.batch}

    def reserve(self, batch: int):
        """Build the work queue for calls with `batch` images (ffst_plan_reserve: allocates and
        synchronises; the transform calls themselves never do).  Done on first use of a batch size."""
        b = int(batch)
        if b not in self._reserved:
            with torch.cuda.device(self.device):
                check(lib.ffst_plan_reserve(self._h, b), "ffst_plan_reserve")
            self._reserved.add(b)

    # -------------------------------------------------------------- buffers
    def empty_coeffs(self, batch: int | None = None):
        b = self.batch if batch is None else batch
        return torch.empty((b, self.eta_local, self.n, self.n), dtype=self.cdtype, device=self.device)

    def empty_images(self, batch: int | None = None):
        b = self.batch if batch is None else batch
        return torch.empty((b, self.n, self.n), dtype=self.dtype, device=self.device)

    def _check_images(self, x):
        if x.dim() == 2:
            x = x.unsqueeze(0)
        if x.dtype != self.dtype or x.device != self.device or x.shape[-2:] != (self.n, self.n):
            raise ValueError(f"images must be {self.dtype} on {self.device} with shape (B, {self.n}, {self.n})")
        if x.shape[0] > self.batch or x.shape[0] < 1:
            raise ValueError(f"batch {x.shape[0]} outside 1..{self.batch}")
        return x.contiguous()

    # -------------------------------------------------------------- transforms
    def forward(self, x, out=None, stream=None, batch: int | None = None):
        """Coefficient cube (B, eta_local, n, n) complex of images x (B, n, n)
        (shearletTransformSpect, eq:shearletTransform).  With a communicator, x is read on rank 0
        only (None elsewhere, with ``batch`` given) and broadcast by the library."""
        if x is None:
            if self.comm is None or self.shard_rank == 0:
                raise ValueError("images required")
            b = self.batch if batch is None else int(batch)
            if b < 1 or b > self.batch:
                raise ValueError(f"batch {b} outside 1..{self.batch}")
            out = self.empty_coeffs(b) if out is None else out
            _check_buf(out, (b, self.eta_local, self.n, self.n), self.cdtype, self.device, "output cube")
            self.reserve(b)
            check(lib.ffst_sheartrans_batch(self._h, None, C.c_void_p(out.data_ptr()), b,
                                            _stream_handle(stream, self.device)), "ffst_sheartrans_batch")
            return out
        x = self._check_images(x)
        b = x.shape[0]
        out = self.empty_coeffs(b) if out is None else out
        _check_buf(out, (b, self.eta_local, self.n, self.n), self.cdtype, self.device, "output cube")
        self.reserve(b)
        check(lib.ffst_sheartrans_batch(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()), b,
                                        _stream_handle(stream, self.device)), "ffst_sheartrans_batch")
        return out

    def inverse(self, c, out=None, stream=None, root: int = 0):
        """Re ifft2(sum_i psi_i fft2(c_i)) (inverseShearletTransformSpect, eq:inverseShearletTransform).
        c: (B, eta_local, n, n) complex.  Sharded with a communicator: the full image, written on
        ``root`` only (the return value elsewhere is an untouched buffer); without one: the
        partial image of the local planes."""
        if c.dim() == 3:
            c = c.unsqueeze(0)
        if c.dtype != self.cdtype or c.device != self.device or c.shape[1:] != (self.eta_local, self.n, self.n):
            raise ValueError("bad coefficient cube")
        c = c.contiguous()
        b = c.shape[0]
        if b < 1 or b > self.batch:
            raise ValueError(f"batch {b} outside 1..{self.batch}")
        out = self.empty_images(b) if out is None else out
        _check_buf(out, (b, self.n, self.n), self.dtype, self.device, "output images")
        self.reserve(b)
        check(lib.ffst_inversesheartrans_batch(self._h, C.c_void_p(c.data_ptr()), C.c_void_p(out.data_ptr()), b,
                                               int(root), _stream_handle(stream, self.device)),
              "ffst_inversesheartrans_batch")
        return out

    def forward_host(self, x_host, out=None, stream=None):
        """Forward from a host (ideally pinned) tensor; the H2D copy runs inside the C call."""
        if x_host.dim() == 2:
            x_host = x_host.unsqueeze(0)
        x_host = x_host.contiguous()
        b = x_host.shape[0]
        if b < 1 or b > self.batch:
            raise ValueError(f"batch {b} outside 1..{self.batch}")
        _check_buf(x_host, (b, self.n, self.n), self.dtype, "cpu", "host images")
        out = self.empty_coeffs(b) if out is None else out
        _check_buf(out, (b, self.eta_local, self.n, self.n), self.cdtype, self.device, "output cube")
        self.reserve(b)
        check(lib.ffst_sheartrans_host(self._h, C.c_void_p(x_host.data_ptr()), C.c_void_p(out.data_ptr()), b,
                                       _stream_handle(stream, self.device)), "ffst_sheartrans_host")
        return out

    def inverse_host(self, c, out_host, stream=None):
        """Inverse into a host (ideally pinned) tensor; the D2H copy runs inside the C call."""
        b = c.shape[0] if c.dim() == 4 else 0
        if b < 1 or b > self.batch:
            raise ValueError(f"batch {b} outside 1..{self.batch}")
        _check_buf(c, (b, self.eta_local, self.n, self.n), self.cdtype, self.device, "coefficient cube")
        _check_buf(out_host, (b, self.n, self.n), self.dtype, "cpu", "host output images")
        self.reserve(b)
        check(lib.ffst_inversesheartrans_host(self._h, C.c_void_p(c.data_ptr()), C.c_void_p(out_host.data_ptr()), b,
                                              _stream_handle(stream, self.device)), "ffst_inversesheartrans_host")
        return out_host

    # -------------------------------------------------------------- compact format (f1)
    def spectra_check(self):
        """(tightness, asymmetry): max |sum_i psi_i^2 - 1| over the grid (the Parseval admission
        check of P:L2219-2220) and max |psi_i(u) - psi_i(-u)| off the Nyquist lines."""
        t, a = C.c_double(), C.c_double()
        check(lib.ffst_plan_spectra_check(self._h, C.byref(t), C.byref(a)), "ffst_plan_spectra_check")
        return t.value, a.value

    def nyquist_planes(self):
        """Local indices of the plan's Nyquist planes (the order of the compact format's G, H)."""
        cnt = C.c_int()
        check(lib.ffst_plan_nyquist_planes(self._h, C.byref(cnt), None), "ffst_plan_nyquist_planes")
        idx = (C.c_int * max(1, cnt.value))()
        check(lib.ffst_plan_nyquist_planes(self._h, C.byref(cnt), idx), "ffst_plan_nyquist_planes")
        return [idx[i] for i in range(cnt.value)]

    def forward_compact(self, x, out=None, gh=None, stream=None):
        """Forward in the compact format: (real parts (B, eta_local, n, n), Nyquist vectors
        gh (B, n_nyq, 2, n)) -- half the bytes of the complex cube, lossless for the forward's
        output (include/ffst.h "compact coefficient format")."""
        x = self._check_images(x)
        b = x.shape[0]
        nn = max(1, len(self.nyquist_planes()))
        out = torch.empty((b, self.eta_local, self.n, self.n), dtype=self.dtype, device=self.device) if out is None else out
        gh = torch.zeros((b, nn, 2, self.n), dtype=self.dtype, device=self.device) if gh is None else gh
        _check_buf(out, (b, self.eta_local, self.n, self.n), self.dtype, self.device, "compact real parts")
        _check_buf(gh, (b, nn, 2, self.n), self.dtype, self.device, "compact Nyquist vectors")
        self.reserve(b)
        check(lib.ffst_sheartrans_compact(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
                                          C.c_void_p(gh.data_ptr()), b, _stream_handle(stream, self.device)),
              "ffst_sheartrans_compact")
        return out, gh

    def inverse_compact(self, re, gh, out=None, stream=None):
        """Inverse from the compact format (see forward_compact)."""
        re = re.contiguous()
        gh = gh.contiguous()
        b = re.shape[0] if re.dim() == 4 else 0
        if b < 1 or b > self.batch:
            raise ValueError(f"batch {b} outside 1..{self.batch}")
        nn = max(1, len(self.nyquist_planes()))
        _check_buf(re, (b, self.eta_local, self.n, self.n), self.dtype, self.device, "compact real parts")
        _check_buf(gh, (b, nn, 2, self.n), self.dtype, self.device, "compact Nyquist vectors")
        out = self.empty_images(b) if out is None else out
        _check_buf(out, (b, self.n, self.n), self.dtype, self.device, "output images")
        self.reserve(b)
        check(lib.ffst_inversesheartrans_compact(self._h, C.c_void_p(re.data_ptr()), C.c_void_p(gh.data_ptr()),
                                                 C.c_void_p(out.data_ptr()), b, _stream_handle(stream, self.device)),
              "ffst_inversesheartrans_compact")
        return out

    def expand_compact(self, re, gh, out=None, stream=None):
        """The complex cube of a compact one: Im c_i(r, m1) = (-1)^r G_i(m1) + (-1)^m1 H_i(r) on the
        Nyquist planes, 0 elsewhere (ffst_expand_compact, one kernel)."""
        b = re.shape[0] if re.dim() == 4 else 0
        if b < 1 or b > self.batch:
            raise ValueError(f"batch {b} outside 1..{self.batch}")
        nn = max(1, len(self.nyquist_planes()))
        _check_buf(re, (b, self.eta_local, self.n, self.n), self.dtype, self.device, "compact real parts")
        _check_buf(gh, (b, nn, 2, self.n), self.dtype, self.device, "compact Nyquist vectors")
        out = self.empty_coeffs(b) if out is None else out
        _check_buf(out, (b, self.eta_local, self.n, self.n), self.cdtype, self.device, "output cube")
        check(lib.ffst_expand_compact(self._h, C.c_void_p(re.data_ptr()), C.c_void_p(gh.data_ptr()),
                                      C.c_void_p(out.data_ptr()), b, _stream_handle(stream, self.device)),
              "ffst_expand_compact")
        return out

    def spectra(self, centred: bool = True, stream=None):
        """The local spectra psi_hat_i as (eta_local, n, n) real (tests / diagnostics)."""
        psi = torch.empty((self.eta_local, self.n, self.n), dtype=self.dtype, device=self.device)
        check(lib.ffst_shearlet_spectra(self._h, C.c_void_p(psi.data_ptr()), int(bool(centred)),
                                        _stream_handle(stream, self.device)), "ffst_shearlet_spectra")
        return psi

    # -------------------------------------------------------------- instrumentation
    def set_timing(self, enable: bool = True):
        check(lib.ffst_plan_set_timing(self._h, int(bool(enable))), "ffst_plan_set_timing")

    def phase_times(self):
        """(fwd_main_ms, inv_main_ms, fwd_total_ms, inv_total_ms), (fwd_launches, inv_launches)."""
        t = (C.c_float * 4)()
        n = (C.c_int * 2)()
        check(lib.ffst_plan_phase_times(self._h, t, n), "ffst_plan_phase_times")
        return tuple(t), tuple(n)

    def set_trace(self, enable: bool = True):
        check(lib.ffst_plan_set_trace(self._h, int(bool(enable))), "ffst_plan_set_trace")

    def trace(self, which: int, batch: int | None = None):
        """Per-item records of the last call: numpy array (items, 10) =
        [type, chunk, smid, t_start, t_ready, t_end, probe0..probe3] (ns)."""
        import numpy as np
        b = self.batch if batch is None else batch
        cap = 1 << 22
        buf = (C.c_ulonglong * (8 * cap))()
        n = C.c_int()
        check(lib.ffst_plan_trace(self._h, int(which), int(b), buf, cap, C.byref(n)), "ffst_plan_trace")
        a = np.ctypeslib.as_array(buf)[: 8 * n.value].reshape(-1, 8).copy()
        out = np.zeros((n.value, 10), dtype=np.int64)
        out[:, 0] = (a[:, 0] >> 32) & 0xFF
        out[:, 1] = a[:, 0] >> 40
        out[:, 2] = a[:, 0] & 0xFFFFFFFF
        out[:, 3:] = a[:, 1:].astype(np.int64)
        return out

    def workspace_bytes(self) -> int:
        v = C.c_size_t()
        check(lib.ffst_plan_workspace_bytes(self._h, C.byref(v)), "ffst_plan_workspace_bytes")
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            lib.ffst_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
