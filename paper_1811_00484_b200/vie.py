"""Host-side mirror of the reference operator API over the C ABI (include/vie_b200.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/vie/{operator,solver}.hpp:
  * ``build_operator_spectra``  operator.hpp:144-177 (from Tucker forms)
  * ``apply_operator``          operator.hpp:273-382 (HosvdDecompress semantics)
  * ``apply_system``            solver.hpp:183-200
  * ``gmres``                   solver.hpp:34-142 (device resident)
``ValueError`` is raised where the reference throws ``std::invalid_argument``.

Device memory and streams come from PyTorch (plumbing only); every number is
computed by libvie_b200.so.  There is no CPU fallback: importing this module
without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VIE_LIB_PATH") or os.path.join(_HERE, "libvie_b200.so")  # override: ablation builds

KIND_N, KIND_K = 0, 1
PWC, PWL = 0, 1
RULE_SIGMA_MAX, RULE_ENERGY = 0, 1

VIE_OK, VIE_EINVAL, VIE_ENOMEM, VIE_ECUDA, VIE_ENCCL = 0, 1, 2, 3, 4

_dp = C.POINTER(C.c_double)
_lib = None

# vie_linear_map_fn / vie_precond (include/vie_b200.h)
_LinearMapFn = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)


class _Precond(C.Structure):
    _fields_ = [("diag", C.c_void_p), ("apply", _LinearMapFn), ("user", C.c_void_p)]


class VieError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[vie error {code}] {msg}")
        self.code = code


def lib() -> C.CDLL:
    """Load libvie_b200.so; fail loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libvie_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
        try:  # torch first: its (newer) NCCL must own libnccl.so.2 before the library pulls it in
            import torch  # noqa: F401
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH)
        L.vie_last_error.restype = C.c_char_p
        L.vie_version.restype = C.c_char_p
        L.vie_system_matvec.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_int,
                                        C.c_void_p]
        L.vie_matvec.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.vie_op_set_strategy.argtypes = [C.c_void_p, C.c_int]
        L.vie_container_info.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.vie_container_read.argtypes = [C.c_char_p, C.c_void_p, C.c_int64]
        L.vie_container_write.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64), C.c_void_p]
        L.vie_tucker_save.argtypes = [C.c_void_p, C.c_char_p]
        L.vie_tucker_load.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]
        L.vie_comm_unique_id.argtypes = [C.c_char_p]
        L.vie_comm_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]
        L.vie_comm_destroy.argtypes = [C.c_void_p]
        L.vie_loopback_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.vie_loopback_destroy.argtypes = [C.c_void_p]
        L.vie_comm_create_loopback.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.vie_op_set_comm.argtypes = [C.c_void_p, C.c_void_p]
        L.vie_slab_matvec.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                      C.c_void_p]
        L.vie_op_get_strategy.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.vie_matvec_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.vie_matvec_host_batch.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.vie_op_set_partition.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.vie_slab_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 4
        L.vie_slab_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.vie_slab_pencil.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.vie_slab_inverse.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                       C.c_int, C.c_void_p]
        L.vie_gmres_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_double,
                                      C.c_int, C.c_int, C.POINTER(_Precond), C.c_void_p, C.POINTER(C.c_int),
                                      C.POINTER(C.c_double), _dp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.c_void_p]
        L.vie_gmres.argtypes = [C.c_void_p, C.c_int64, _LinearMapFn, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                C.c_int, C.c_int, C.POINTER(_Precond), C.c_void_p, C.POINTER(C.c_int),
                                C.POINTER(C.c_double), _dp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.c_void_p]
        L.vie_matvec_timed.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != VIE_OK:
        msg = lib().vie_last_error().decode()
        if rc == VIE_EINVAL:
            raise ValueError(msg)
        raise VieError(rc, msg)


def _i64(vals):
    return (C.c_int64 * len(vals))(*[int(v) for v in vals])


def _cplx(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def component_table(kind: int, basis: int):
    """Canonical components/parities/blocks of (kind, basis) from the product library."""
    nc, nb = C.c_int(), C.c_int()
    comps = (C.c_int * 256)()
    par = (C.c_int * 192)()
    blocks = (C.c_int * 1024)()
    _check(lib().vie_component_table(int(kind), int(basis), C.byref(nc), comps, par, C.byref(nb), blocks))
    return (np.array(comps[: 4 * nc.value], np.int32).reshape(-1, 4),
            np.array(par[: 3 * nc.value], np.int32).reshape(-1, 3),
            np.array(blocks[: 4 * nb.value], np.int32).reshape(-1, 4))


def ncur(basis: int) -> int:
    return 3 if basis == PWC else 12


class DftService:
    """Context: CUDA device + stream + FFT plan cache (fft.hpp DftService)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().vie_ctx_create(C.byref(self._h), int(device)))
        self.device = device

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        _check(lib().vie_ctx_sync(self._h))

    def close(self):
        if self._h:
            lib().vie_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TuckerForm:
    """Device-resident Fourier-domain Tucker form of one component."""

    def __init__(self, dft: DftService, dims, core, factors: Sequence, sign, domain: int = 0):
        core = _cplx(np.asarray(core).reshape(-1, order="F"))
        us = [np.asfortranarray(np.asarray(u, np.complex128)) for u in factors]
        ranks = [u.shape[1] for u in us]
        if core.size != ranks[0] * ranks[1] * ranks[2]:
            raise ValueError("TuckerForm: core size does not match the factor ranks")
        rows = [d if domain == 0 else 2 * d for d in dims]
        for q in range(3):
            if us[q].shape[0] != rows[q]:
                raise ValueError("TuckerForm: factor rows do not match dims")
        self._h = C.c_void_p()
        self._dft = dft
        _check(lib().vie_tucker_from_factors(dft.handle, _i64(dims), _i64(ranks), core.ctypes.data_as(_dp),
                                             us[0].ctypes.data_as(_dp), us[1].ctypes.data_as(_dp),
                                             us[2].ctypes.data_as(_dp), (C.c_int * 3)(*[int(s) for s in sign]),
                                             int(domain), C.byref(self._h)))
        self.dims = tuple(int(d) for d in dims)
        self.ranks = tuple(ranks)
        self.sign = tuple(int(s) for s in sign)

    @property
    def handle(self):
        return self._h

    @classmethod
    def _from_handle(cls, dft, h, dims, ranks, sign):
        obj = cls.__new__(cls)
        obj._h, obj._dft = h, dft
        obj.dims, obj.ranks, obj.sign = tuple(dims), tuple(ranks), tuple(sign)
        return obj

    def __del__(self):
        try:
            if self._h:
                lib().vie_tucker_destroy(self._h)
        except Exception:
            pass


def tucker_cp_form(dft: DftService, dims, factors: Sequence, sign, domain: int = 0) -> TuckerForm:
    """TuckerCPForm (decomp.hpp:143-148; merged factors W_q, n_q x R) on the device
    (vie_tucker_from_cp): served by the fused matvec as the Tucker form with the
    superdiagonal R^3 core, i.e. the TuckerCpLoop / decompress_cp spectrum
    (operator.hpp:248-261, 346-362)."""
    ws = [np.asfortranarray(np.asarray(w, np.complex128)) for w in factors]
    rank = ws[0].shape[1]
    if any(w.shape[1] != rank for w in ws):
        raise ValueError("TuckerCPForm: factor column counts differ")
    rows = [d if domain == 0 else 2 * d for d in dims]
    if any(ws[q].shape[0] != rows[q] for q in range(3)):
        raise ValueError("TuckerCPForm: factor rows do not match dims")
    h = C.c_void_p()
    _check(lib().vie_tucker_from_cp(dft.handle, _i64(dims), C.c_int64(rank), ws[0].ctypes.data_as(_dp),
                                    ws[1].ctypes.data_as(_dp), ws[2].ctypes.data_as(_dp),
                                    (C.c_int * 3)(*[int(x) for x in sign]), int(domain), C.byref(h)))
    return TuckerForm._from_handle(dft, h, dims, (rank,) * 3, sign)


# ----------------------------------------------------------------------------- VIET container
CONTAINER_DENSE, CONTAINER_TUCKER, CONTAINER_TUCKER_CP = 0, 1, 2


def _path(p) -> bytes:
    import os

    return os.fsencode(p)


def container_info(path) -> dict:
    """Header of a VIET file (container.hpp:15-29): kind, rule, tol, dims, ranks."""
    k, r, t = C.c_int(), C.c_int(), C.c_double()
    d, rk = (C.c_int64 * 3)(), (C.c_int64 * 3)()
    _check(lib().vie_container_info(_path(path), C.byref(k), C.byref(r), C.byref(t), d, rk))
    return {"kind": k.value, "rule": r.value, "tol": t.value, "dims": tuple(d), "ranks": tuple(rk)}


def save_container(path, value, dims=None) -> None:
    """save_container (container.hpp:95-123).  value: a 3-D complex array (dense Tensor3,
    axis-1 fastest: pass it in (n1, n2, n3) Fortran order or as a flat reference-layout
    vector with `dims`), a device TuckerForm built from spatial factors (tucker_compress,
    TuckerForm(domain=0), tucker_cp_form), or a host tuple ("tucker", core, (U1, U2, U3),
    rule, tol) / ("tucker_cp", (W1, W2, W3))."""
    if isinstance(value, TuckerForm):
        _check(lib().vie_tucker_save(value.handle, _path(path)))
        return
    if isinstance(value, tuple) and value and value[0] in ("tucker", "tucker_cp"):
        if value[0] == "tucker":
            _, core, us, rule, tol = value
            us = [np.asfortranarray(np.asarray(u, np.complex128)) for u in us]
            ranks = [u.shape[1] for u in us]
            payload = np.concatenate([u.reshape(-1, order="F") for u in us] +
                                     [_cplx(np.asarray(core).reshape(-1, order="F"))])
            kind, rr, tt = CONTAINER_TUCKER, int(rule), float(tol)
        else:
            ws = [np.asfortranarray(np.asarray(w, np.complex128)) for w in value[1]]
            ranks = [ws[0].shape[1]] * 3
            payload = np.concatenate([w.reshape(-1, order="F") for w in ws])
            kind, rr, tt = CONTAINER_TUCKER_CP, 0, 0.0
        d = [u.shape[0] for u in (us if kind == CONTAINER_TUCKER else ws)]
        _check(lib().vie_container_write(_path(path), kind, rr, tt, _i64(d), _i64(ranks),
                                         np.ascontiguousarray(payload).ctypes.data))
        return
    a = np.asarray(value, np.complex128)
    if a.ndim == 3:
        d, flat = a.shape, a.reshape(-1, order="F")
    else:
        if dims is None:
            raise ValueError("save_container: dims needed for a flat tensor")
        d, flat = tuple(dims), a.reshape(-1)
    flat = np.ascontiguousarray(flat)
    _check(lib().vie_container_write(_path(path), CONTAINER_DENSE, 0, 0.0, _i64(d), _i64([0, 0, 0]),
                                     flat.ctypes.data))


def load_container(path, dft: DftService | None = None, sign=None):
    """load_container (container.hpp:125-159).  Dense files give a (n1, n2, n3) complex array
    (Fortran order, axis-1 fastest).  Compressed forms give a device TuckerForm when `dft`
    and the component parity `sign` are passed, else the host tuple of save_container."""
    info = container_info(path)
    if info["kind"] != CONTAINER_DENSE and dft is not None:
        if sign is None:
            raise ValueError("load_container: the component parity `sign` is needed for a device form")
        h = C.c_void_p()
        _check(lib().vie_tucker_load(dft.handle, _path(path), (C.c_int * 3)(*[int(x) for x in sign]), C.byref(h)))
        return TuckerForm._from_handle(dft, h, info["dims"], info["ranks"], sign)
    d, rk = info["dims"], info["ranks"]
    n = int(np.prod(d)) if info["kind"] == CONTAINER_DENSE else \
        sum(d[q] * rk[q] for q in range(3)) + (int(np.prod(rk)) if info["kind"] == CONTAINER_TUCKER else 0)
    buf = np.empty(n, np.complex128)
    _check(lib().vie_container_read(_path(path), buf.ctypes.data, n))
    if info["kind"] == CONTAINER_DENSE:
        return buf.reshape(d, order="F")
    mats, off = [], 0
    for q in range(3):
        mats.append(buf[off:off + d[q] * rk[q]].reshape(d[q], rk[q], order="F"))
        off += d[q] * rk[q]
    if info["kind"] == CONTAINER_TUCKER_CP:
        return ("tucker_cp", tuple(mats))
    return ("tucker", buf[off:].reshape(rk, order="F"), tuple(mats), info["rule"], info["tol"])


def tucker_compress(dft: DftService, t, dims, sign, tol: float = 1e-8, rule: int = RULE_ENERGY) -> TuckerForm:
    """hosvd + transform_factors (decomp.hpp:160-176, operator.hpp:76-90) of a spatial
    Toeplitz-defining tensor (flat, reference layout; host array or CUDA tensor, the
    latter compressed in place on the device); returns the device form."""
    if hasattr(t, "is_cuda") and t.is_cuda:
        torch = _torch()
        tt = t.reshape(-1).to(torch.complex128).contiguous()
        if tt.numel() != int(np.prod(dims)):
            raise ValueError("tucker_compress: tensor size does not match dims")
        h = C.c_void_p()
        ranks = (C.c_int64 * 3)()
        _check(lib().vie_tucker_compress_device(dft.handle, _i64(dims), C.c_void_p(tt.data_ptr()),
                                                (C.c_int * 3)(*[int(x) for x in sign]), C.c_double(tol), int(rule),
                                                C.byref(h), ranks, C.c_void_p(_stream_handle(None, tt.device))))
        return TuckerForm._from_handle(dft, h, dims, [ranks[0], ranks[1], ranks[2]], sign)
    t = _cplx(np.asarray(t).reshape(-1, order="F") if np.asarray(t).ndim == 3 else t).reshape(-1)
    if t.size != int(np.prod(dims)):
        raise ValueError("tucker_compress: tensor size does not match dims")
    h = C.c_void_p()
    ranks = (C.c_int64 * 3)()
    _check(lib().vie_tucker_compress(dft.handle, _i64(dims), t.ctypes.data_as(_dp),
                                     (C.c_int * 3)(*[int(x) for x in sign]), C.c_double(tol), int(rule),
                                     C.byref(h), ranks))
    return TuckerForm._from_handle(dft, h, dims, [ranks[0], ranks[1], ranks[2]], sign)


@dataclass
class CpAlsResult:
    """CpAlsResult (decomp.hpp:184-190): factors (dims[q], r), error per sweep, flags."""
    factors: list
    rel_error_trace: np.ndarray
    converged: bool
    ill_posed_rank: bool


def cp_als(t, dims, r: int, max_iters: int = 100, stall_tol: float = 1e-12, seed: int = 0x5EED) -> CpAlsResult:
    """cp_als (decomp.hpp:237-298) of a host tensor (flat, reference layout): the CP fitting
    of a Tucker core (r1 r2 r3 entries), run by the library next to the HOSVD's r x r
    eigenproblems (cp_als.cu)."""
    t = _cplx(np.asarray(t).reshape(-1, order="F") if np.asarray(t).ndim == 3 else t).reshape(-1)
    if t.size != int(np.prod(dims)):
        raise ValueError("cp_als: tensor size does not match dims")
    if r < 0:
        raise ValueError("cp_als: rank must be >= 0")
    fs = [np.zeros(max(int(dims[q]) * int(r), 1), np.complex128) for q in range(3)]
    cap = max(int(max_iters), 1) + 1
    tr = np.empty(cap)
    nt = C.c_int()
    flags = (C.c_int * 2)()
    _check(lib().vie_cp_als(_i64(dims), t.ctypes.data_as(_dp), C.c_int64(r), int(max_iters), C.c_double(stall_tol),
                            C.c_uint64(seed), fs[0].ctypes.data_as(_dp), fs[1].ctypes.data_as(_dp),
                            fs[2].ctypes.data_as(_dp), tr.ctypes.data_as(_dp), cap, C.byref(nt), flags))
    facs = [fs[q][:int(dims[q]) * int(r)].reshape((int(dims[q]), int(r)), order="F") for q in range(3)]
    return CpAlsResult(facs, tr[:nt.value].copy(), bool(flags[0]), bool(flags[1]))


@dataclass
class TuckerCpResult:
    """TuckerCpResult (decomp.hpp:300-307): `form` is the device form of
    transform_factors(TuckerCPForm) (operator.hpp:92-106), `factors` the spatial merged
    factors W_q = U_q V_q."""
    form: "TuckerForm"
    factors: list
    rank: int
    hosvd_relative_error: float
    core_cp_relative_error: float
    achieved_relative_error: float
    cp_error_trace: np.ndarray


def tucker_cp(dft: DftService, t, dims, sign, tol: float, cp_iters: int = 1000, rule: int = RULE_ENERGY,
              cp_rank: int = -1, stall_tol: float = 0.0) -> TuckerCpResult:
    """tucker_cp (decomp.hpp:336-373): HOSVD on the device, CP-ALS on the core, merged
    factors; t is a host array or a CUDA tensor (flat, reference layout)."""
    on_dev = hasattr(t, "is_cuda") and t.is_cuda
    if on_dev:
        tt = t.reshape(-1).to(_torch().complex128).contiguous()
        ptr, n = C.c_void_p(tt.data_ptr()), tt.numel()
        stream = C.c_void_p(_stream_handle(None, tt.device))
    else:
        tt = _cplx(np.asarray(t).reshape(-1, order="F") if np.asarray(t).ndim == 3 else t).reshape(-1)
        ptr, n, stream = C.c_void_p(tt.ctypes.data), tt.size, None
    if n != int(np.prod(dims)):
        raise ValueError("tucker_cp: tensor size does not match dims")
    cap = int(cp_rank) if cp_rank >= 0 else int(min(dims))
    ws = [np.zeros(max(int(dims[q]) * cap, 1), np.complex128) for q in range(3)]
    h = C.c_void_p()
    rk = C.c_int64()
    errs = (C.c_double * 3)()
    trc = int(cp_iters) + 1
    tr = np.empty(trc)
    nt = C.c_int()
    _check(lib().vie_tucker_cp(dft.handle, _i64(dims), ptr, int(on_dev), (C.c_int * 3)(*[int(x) for x in sign]),
                               C.c_double(tol), int(rule), int(cp_iters), C.c_int64(cp_rank), C.c_double(stall_tol),
                               C.byref(h), C.byref(rk), ws[0].ctypes.data_as(_dp), ws[1].ctypes.data_as(_dp),
                               ws[2].ctypes.data_as(_dp), C.c_int64(cap), errs, tr.ctypes.data_as(_dp), trc,
                               C.byref(nt), stream))
    r = rk.value
    form = TuckerForm._from_handle(dft, h, dims, (r,) * 3, sign)
    facs = [ws[q][:int(dims[q]) * r].reshape((int(dims[q]), r), order="F") for q in range(3)]
    return TuckerCpResult(form, facs, r, errs[0], errs[1], errs[2], tr[:nt.value].copy())


@dataclass
class EmbeddedSpectrum:
    """Device operator (operator.hpp:120-129) holding Tucker forms only."""
    kind: int
    basis: int
    grid_dims: tuple
    handle: C.c_void_p
    dft: DftService
    comps: list = field(default_factory=list)
    local_elems: int | None = None  # slab-partitioned: this rank's z-slab size (sharding.SlabMatvec)

    @property
    def embedded_dims(self):
        return tuple(2 * d for d in self.grid_dims)

    @property
    def n_cur(self) -> int:
        return ncur(self.basis)

    @property
    def n_vox(self) -> int:
        return int(np.prod(self.grid_dims))

    def workspace_bytes(self) -> int:
        ws = C.c_int64()
        _check(lib().vie_op_info(self.handle, None, None, C.byref(ws)))
        return ws.value

    def set_profiling(self, on):
        """True/1: serial stages with per-kernel event times; 2: the overlapped schedule with
        events after the forward passes, after the decompression join and at the end."""
        _check(lib().vie_op_set_profiling(self.handle, 2 if on == 2 else int(bool(on))))

    def last_stats(self):
        n = C.c_int()
        ms = (C.c_double * 8)()
        _check(lib().vie_op_last_stats(self.handle, C.byref(n), ms))
        return n.value, list(ms)

    def close(self):
        if self.handle:
            lib().vie_op_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_operator_spectra(kind: int, basis: int, grid, comps: Sequence, forms: Sequence[TuckerForm],
                           dft: DftService) -> EmbeddedSpectrum:
    """operator.hpp:144-177 from compressed forms; comps[i] = (q, q', l, l')."""
    comps = [tuple(int(v) for v in c) for c in comps]
    if len(comps) == 0:
        raise ValueError("build_operator_spectra: no components")
    if len(comps) != len(forms):
        raise ValueError("build_operator_spectra: one form per component required")
    flat = (C.c_int * (4 * len(comps)))(*[v for c in comps for v in c])
    hs = (C.c_void_p * len(forms))(*[f.handle.value for f in forms])
    h = C.c_void_p()
    _check(lib().vie_op_create(dft.handle, int(kind), int(basis), _i64(grid), len(comps), flat, hs, C.byref(h)))
    return EmbeddedSpectrum(int(kind), int(basis), tuple(int(g) for g in grid), h, dft, comps)


# ----------------------------------------------------------------------------- apply
def _torch():
    import torch
    return torch


def _stream_handle(stream, device):
    """CUDA stream handle for the C ABI.  torch's default stream has handle 0,
    which the C ABI reads as 'context stream'; map it to cudaStreamLegacy (1)
    so kernels order with torch work on the default stream."""
    if stream is None:
        stream = _torch().cuda.current_stream(device).cuda_stream
    return stream if stream else 1


def _dev_vec(op: EmbeddedSpectrum, x):
    torch = _torch()
    n = op.local_elems if op.local_elems is not None else op.n_cur * op.n_vox
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise TypeError("expected a CUDA torch.complex128 tensor")
    if x.dtype != torch.complex128 or x.numel() != n:
        raise ValueError("apply_operator: dim mismatch")
    return x.contiguous()


COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    """NCCL unique id for a new communicator (vie_comm_unique_id); rank 0 creates it and the
    caller broadcasts the bytes."""
    buf = C.create_string_buffer(COMM_ID_BYTES)
    _check(lib().vie_comm_unique_id(buf))
    return buf.raw


class Loopback:
    """Shared state of a loopback transport (vie_loopback_create): `world` ranks of this process,
    one host thread each, exchanging by device copies between host barriers (tests)."""

    def __init__(self, world: int):
        self.world = world
        self.handle = C.c_void_p()
        _check(lib().vie_loopback_create(int(world), C.byref(self.handle)))

    def __del__(self):
        try:
            if self.handle:
                lib().vie_loopback_destroy(self.handle)
                self.handle = C.c_void_p()
        except Exception:
            pass


class Comm:
    """Communicator of the library over `world` ranks: NCCL (vie_comm_create, one process per
    GPU) or, with `loopback`, the test transport (vie_comm_create_loopback)."""

    def __init__(self, dft: DftService, world: int, rank: int, uid: bytes | None = None,
                 loopback: Loopback | None = None):
        self.world, self.rank, self.dft, self._lb = world, rank, dft, loopback
        self.handle = C.c_void_p()
        if loopback is not None:
            if loopback.world != world:
                raise ValueError("Comm: loopback size differs from world")
            _check(lib().vie_comm_create_loopback(dft.handle, loopback.handle, int(rank), C.byref(self.handle)))
            return
        if uid is None or len(uid) != COMM_ID_BYTES:
            raise ValueError("Comm: unique id must be COMM_ID_BYTES bytes")
        _check(lib().vie_comm_create(dft.handle, int(world), int(rank), uid, C.byref(self.handle)))

    def __del__(self):
        try:
            if self.handle:
                lib().vie_comm_destroy(self.handle)
                self.handle = C.c_void_p()
        except Exception:
            pass


def set_strategy(op: EmbeddedSpectrum, strategy: str) -> None:
    """Strategy of every later apply on ``op`` (vie_op_set_strategy): 'hosvd_decompress' /
    'tucker_cp_decompress' or 'hosvd_loop' / 'tucker_cp_loop'."""
    codes = {"hosvd_decompress": 1, "tucker_cp_decompress": 1, "hosvd_loop": 2, "tucker_cp_loop": 2}
    if strategy not in codes:
        raise ValueError(f"set_strategy: unknown strategy {strategy!r}")
    _check(lib().vie_op_set_strategy(op.handle, codes[strategy]))


def get_strategy(op: EmbeddedSpectrum) -> str:
    v = C.c_int()
    _check(lib().vie_op_get_strategy(op.handle, C.byref(v)))
    return "hosvd_loop" if v.value == 2 else "hosvd_decompress"


def apply_operator(op: EmbeddedSpectrum, x, strategy: str | None = None, policy: str = "with_buffer",
                   ws=None, dft=None, out=None, stream=None):
    """y = A x (operator.hpp:273).  ``x``: CUDA complex128 tensor (S*N_v) or host numpy array.

    Strategies (operator.hpp:17-31): 'hosvd_decompress' decompresses every component's octant
    spectrum into one HBM buffer read by the fused axis-3 FFT x Hadamard pass; 'hosvd_loop' is
    the buffer-free form -- one persistent kernel decompresses spectrum tiles into an
    L2-resident ring and consumes them (PWL, ranks <= 28; ValueError otherwise).  The
    'tucker_cp_*' names select the same two paths (CP forms are held as Tucker forms).  The
    reference's scratch-policy contract is kept: decompress strategies with policy
    'no_buffer' raise ValueError (operator.hpp:278-281).  The strategy sticks to the operator
    (vie_op_set_strategy) for later system matvecs and solves; strategy=None keeps it."""
    loop = {"hosvd_decompress": False, "tucker_cp_decompress": False, "hosvd_loop": True, "tucker_cp_loop": True}
    if strategy is None:  # the operator's current strategy (hosvd_decompress unless set)
        strategy = get_strategy(op)
    if strategy not in loop:
        raise ValueError(f"apply_operator: strategy {strategy!r} needs a representation this build does not hold")
    if not loop[strategy] and policy == "no_buffer":
        raise ValueError("apply_operator: decompress strategies need ScratchPolicy::WithBuffer")
    set_strategy(op, strategy)
    if isinstance(x, np.ndarray):
        xa = _cplx(x).reshape(-1)
        if xa.size != op.n_cur * op.n_vox:
            raise ValueError("apply_operator: dim mismatch")
        y = np.empty_like(xa)
        _check(lib().vie_matvec_host(op.handle, xa.ctypes.data, y.ctypes.data))
        return y
    torch = _torch()
    x = _dev_vec(op, x)
    y = out if out is not None else torch.empty_like(x)
    _check(lib().vie_matvec(op.handle, x.data_ptr(), y.data_ptr(), _stream_handle(stream, x.device)))
    return y


def apply_operator_batch(op: EmbeddedSpectrum, xs, ys=None):
    """Independent applications y_i = A x_i of HOST vectors (numpy complex128 or CPU
    torch tensors, pinned for copy/compute overlap), pipelined on the device
    (vie_matvec_host_batch): the copies of neighbouring vectors overlap each matvec."""
    xs = list(xs)
    n = op.n_cur * op.n_vox
    ptr = lambda a: a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
    for x in xs:
        if (x.numel() if hasattr(x, "numel") else x.size) != n:
            raise ValueError("apply_operator: dim mismatch")
    if ys is None:
        ys = [np.empty(n, dtype=np.complex128) for _ in xs]
    if len(ys) != len(xs):
        raise ValueError("apply_operator: dim mismatch")
    xp = (C.c_void_p * max(1, len(xs)))(*[ptr(x) for x in xs])
    yp = (C.c_void_p * max(1, len(ys)))(*[ptr(y) for y in ys])
    _check(lib().vie_matvec_host_batch(op.handle, len(xs), xp, yp))
    return ys


def apply_system(eps_r, inv_v: float, op: EmbeddedSpectrum, x, out=None, diag_term: bool = True, stream=None):
    """y = eps*g*x - (eps-1)*inv_v*(N x) (solver.hpp:183-200); CUDA tensors."""
    torch = _torch()
    x = _dev_vec(op, x)
    if not (isinstance(eps_r, torch.Tensor) and eps_r.is_cuda and eps_r.numel() == op.n_vox):
        raise ValueError("apply_system: dim mismatch")
    eps_r = eps_r.to(torch.complex128).contiguous()
    y = out if out is not None else torch.empty_like(x)
    _check(lib().vie_system_matvec(op.handle, eps_r.data_ptr(), float(inv_v), x.data_ptr(), y.data_ptr(),
                                   int(bool(diag_term)), _stream_handle(stream, x.device)))
    return y


@dataclass
class GmresConfig:  # solver.hpp:12-16
    tolerance: float = 1e-5
    inner: int = 50
    outer: int = 200


@dataclass
class GmresResult:  # solver.hpp:18-24
    solution: object
    residual_history: list
    final_relative_residual: float
    iterations: int
    converged: bool


class _DevView:
    """Zero-copy view of n complex128 values at a device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _map_callback(fn, n: int, device):
    """C callback for a Python device map fn(x, y) (torch CUDA tensors), run on the
    solve's stream."""
    torch = _torch()

    def cb(user, xp, yp, stream):
        x = torch.as_tensor(_DevView(xp, n), device=device)
        y = torch.as_tensor(_DevView(yp, n), device=device)
        with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=device)):
            fn(x, y)

    return _LinearMapFn(cb)


def _precond_struct(precond, n: int, device):
    """None -> no preconditioner; CUDA tensor of n values -> diagonal M; callable
    fn(x, y) -> the callback form.  Returns (struct or None, keep-alive)."""
    torch = _torch()
    if precond is None:
        return None, None
    if isinstance(precond, torch.Tensor):
        if not (precond.is_cuda and precond.numel() == n):
            raise ValueError("gmres: diagonal preconditioner must be a CUDA tensor of n values")
        d = precond.to(torch.complex128).contiguous()
        return _Precond(d.data_ptr(), _LinearMapFn(), None), d
    if callable(precond):
        cb = _map_callback(precond, n, device)
        return _Precond(None, cb, None), cb
    raise ValueError("gmres: precond must be None, a CUDA tensor or a callable")


def gmres(op: EmbeddedSpectrum, eps_r, inv_v: float, rhs, cfg: GmresConfig = GmresConfig(), x0=None,
          history_cap: int = 100000, precond=None, stream=None) -> GmresResult:
    """Restarted GMRES on apply_system, device resident (solver.hpp:34-142); optional
    right preconditioner (solver.hpp:74, :131): a CUDA tensor (diagonal) or fn(x, y)."""
    torch = _torch()
    rhs = _dev_vec(op, rhs)
    eps_r = eps_r.to(torch.complex128).contiguous()
    x = torch.empty_like(rhs)
    x0p = _dev_vec(op, x0).data_ptr() if x0 is not None else None
    pc, keep = _precond_struct(precond, rhs.numel(), rhs.device)
    it, hl, cv = C.c_int(), C.c_int(), C.c_int()
    fr = C.c_double()
    hist = np.empty(history_cap, np.float64)
    _check(lib().vie_gmres_solve(op.handle, eps_r.data_ptr(), float(inv_v), rhs.data_ptr(), x0p,
                                 float(cfg.tolerance), int(cfg.inner), int(cfg.outer),
                                 C.byref(pc) if pc is not None else None, x.data_ptr(),
                                 C.byref(it), C.byref(fr), hist.ctypes.data_as(_dp), int(history_cap),
                                 C.byref(hl), C.byref(cv), _stream_handle(stream, rhs.device)))
    del keep
    return GmresResult(x, hist[: min(hl.value, history_cap)].tolist(), fr.value, it.value, bool(cv.value))


def gmres_map(dft: DftService, apply, rhs, cfg: GmresConfig = GmresConfig(), x0=None, precond=None,
              history_cap: int = 100000) -> GmresResult:
    """gmres(apply, rhs, cfg, x0, precond) of solver.hpp:34 for any device linear map
    apply(x, y) (y = A x, torch CUDA complex128 tensors), on the device GMRES (vie_gmres)."""
    torch = _torch()
    if not (isinstance(rhs, torch.Tensor) and rhs.is_cuda and rhs.dtype == torch.complex128):
        raise ValueError("gmres: rhs must be a CUDA complex128 tensor")
    rhs = rhs.contiguous()
    n = rhs.numel()
    if x0 is not None and x0.numel() != n:
        raise ValueError("gmres: initial guess size mismatch")
    x = torch.empty_like(rhs)
    x0c = x0.to(torch.complex128).contiguous() if x0 is not None else None
    cb = _map_callback(apply, n, rhs.device)
    pc, keep = _precond_struct(precond, n, rhs.device)
    it, hl, cv = C.c_int(), C.c_int(), C.c_int()
    fr = C.c_double()
    hist = np.empty(history_cap, np.float64)
    _check(lib().vie_gmres(dft.handle, n, cb, None, rhs.data_ptr(), x0c.data_ptr() if x0c is not None else None,
                           float(cfg.tolerance), int(cfg.inner), int(cfg.outer),
                           C.byref(pc) if pc is not None else None, x.data_ptr(), C.byref(it), C.byref(fr),
                           hist.ctypes.data_as(_dp), int(history_cap), C.byref(hl), C.byref(cv),
                           _stream_handle(None, rhs.device)))
    del keep, cb
    return GmresResult(x, hist[: min(hl.value, history_cap)].tolist(), fr.value, it.value, bool(cv.value))


@dataclass
class ApplyTimings:  # operator.hpp:189-192
    fft_ms: float = 0.0
    product_ms: float = 0.0


def apply_operator_timed(op: EmbeddedSpectrum, x, timings: ApplyTimings, out=None):
    """apply_operator with ApplyTimings (vie_matvec_timed): serialised stages, CUDA events."""
    torch = _torch()
    x = _dev_vec(op, x)
    y = out if out is not None else torch.empty_like(x)
    torch.cuda.current_stream(x.device).synchronize()
    f, p = C.c_double(), C.c_double()
    _check(lib().vie_matvec_timed(op.handle, x.data_ptr(), y.data_ptr(), C.byref(f), C.byref(p)))
    timings.fft_ms, timings.product_ms = f.value, p.value
    return y


# ----------------------------------------------------------------------------- assembly
KIND_G = 2  # OperatorKind::ScalarG


@dataclass
class QuadratureSpec:  # assembly.hpp:24-36
    far_points_per_axis: int = 5
    near_points_per_axis: int = 10
    near_radius: int = 1
    surface_points_per_axis: int = 12
    volume_points_per_axis: int = 6


class _Quad(C.Structure):  # vie_quadrature
    _fields_ = [("far", C.c_int), ("near", C.c_int), ("near_radius", C.c_int), ("surface", C.c_int),
                ("volume", C.c_int)]


def _quad(q: "QuadratureSpec | None"):
    q = q or QuadratureSpec()
    return _Quad(q.far_points_per_axis, q.near_points_per_axis, q.near_radius, q.surface_points_per_axis,
                 q.volume_points_per_axis)


def assemble_defining_tensor(dft: DftService, grid: "VoxelGrid", k0: float, kind: int, row_axis: int, col_axis: int,
                             quad: "QuadratureSpec | None" = None, basis: int = PWC):
    """assemble_defining_tensor (assembly.hpp:159-233) on the device: the PWC Galerkin
    Toeplitz-defining tensor of one component; CUDA complex128 tensor (flat, reference layout)."""
    torch = _torch()
    nv = int(np.prod(grid.dims))
    t = torch.empty(nv, dtype=torch.complex128, device=f"cuda:{dft.device}")
    qs = _quad(quad)
    _check(lib().vie_assemble(dft.handle, _i64(grid.dims), (C.c_double * 3)(*[float(r) for r in grid.resolution]),
                              C.c_double(k0), int(kind), int(row_axis), int(col_axis), int(basis), C.byref(qs),
                              C.c_void_p(t.data_ptr()), C.c_void_p(_stream_handle(None, t.device))))
    return t


def assemble_operator(dft: DftService, grid: "VoxelGrid", k0: float, kind: int,
                      quad: "QuadratureSpec | None" = None):
    """assemble_operator (assembly.hpp:236-244): [(component (q, q', 0, 0), tensor)] over the
    unique PWC components of kind N or K (components.hpp:71-92), on the device."""
    comps, _, _ = component_table(kind, PWC)
    return [(tuple(int(v) for v in c), assemble_defining_tensor(dft, grid, k0, kind, int(c[0]), int(c[1]), quad))
            for c in comps]


def self_static_term(dft: DftService, delta, quad: "QuadratureSpec | None" = None):
    """self_static_term (assembly.hpp:127-150): (dyad diagonal, gram, error indicator, converged)."""
    dg = (C.c_double * 3)()
    gram, err, conv = C.c_double(), C.c_double(), C.c_int()
    qs = _quad(quad)
    _check(lib().vie_self_static_term(dft.handle, (C.c_double * 3)(*[float(d) for d in delta]), C.byref(qs), dg,
                                      C.byref(gram), C.byref(err), C.byref(conv)))
    return np.array(dg[:]), gram.value, err.value, bool(conv.value)


# ----------------------------------------------------------------------------- scene stages
@dataclass
class VoxelGrid:  # grid.hpp:24-46
    dims: tuple
    resolution: tuple = (1.0, 1.0, 1.0)
    origin: tuple = (0.0, 0.0, 0.0)

    def voxel_volume(self) -> float:
        return float(self.resolution[0] * self.resolution[1] * self.resolution[2])


@dataclass
class DielectricMap:  # grid.hpp:52-75; eps_r: CUDA complex128 tensor of n_vox (flat = i + n1 (j + n2 k))
    grid: VoxelGrid
    eps_r: object
    frequency: float


@dataclass
class PlaneWave:  # grid.hpp:78-100 (normalised and checked by the library)
    polarization: tuple = (1.0, 0.0, 0.0)
    direction: tuple = (0.0, 0.0, 1.0)
    amplitude: float = 1.0


class _Scene(C.Structure):  # vie_scene (include/vie_b200.h)
    _fields_ = [("dims", C.c_int64 * 3), ("resolution", C.c_double * 3), ("origin", C.c_double * 3),
                ("frequency", C.c_double), ("polarization", C.c_double * 3), ("direction", C.c_double * 3),
                ("amplitude", C.c_double)]


def _scene(m: DielectricMap, inc: PlaneWave | None) -> _Scene:
    inc = inc or PlaneWave()
    return _Scene((C.c_int64 * 3)(*[int(v) for v in m.grid.dims]),
                  (C.c_double * 3)(*[float(v) for v in m.grid.resolution]),
                  (C.c_double * 3)(*[float(v) for v in m.grid.origin]), float(m.frequency),
                  (C.c_double * 3)(*[float(v) for v in inc.polarization]),
                  (C.c_double * 3)(*[float(v) for v in inc.direction]), float(inc.amplitude))


def _eps_dev(m: DielectricMap):
    torch = _torch()
    nv = int(np.prod(m.grid.dims))
    e = m.eps_r
    if not (isinstance(e, torch.Tensor) and e.is_cuda and e.numel() == nv):
        raise ValueError("DielectricMap: eps_r must be a CUDA tensor of n_vox values")
    return e.to(torch.complex128).contiguous()


def _field_dev(x, nv: int, what: str):
    torch = _torch()
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.complex128 and x.numel() == 3 * nv):
        raise ValueError(f"{what}: expected a CUDA complex128 PWC field of 3 n_vox values")
    return x.contiguous()


def build_rhs(m: DielectricMap, inc: PlaneWave, quad_points_per_axis: int = 1, stream=None):
    """build_rhs (solver.hpp:148-179) on the device: 3 n_vox complex (PWC)."""
    torch = _torch()
    eps = _eps_dev(m)
    sc = _scene(m, inc)
    out = torch.empty(3 * eps.numel(), dtype=torch.complex128, device=eps.device)
    with torch.cuda.device(eps.device):
        _check(lib().vie_build_rhs(None, C.byref(sc), C.c_void_p(eps.data_ptr()), C.c_int(int(quad_points_per_axis)),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(_stream_handle(stream, eps.device))))
    return out


@dataclass
class Fields:  # solver.hpp:202-206
    e: object
    h: object = None
    has_h: bool = False


def recover_fields(j, m: DielectricMap, inc: PlaneWave, op_k: "EmbeddedSpectrum | None" = None, stream=None) -> Fields:
    """recover_fields (solver.hpp:211-249): e from j (incident field where chi_e = 0);
    h = h_inc + K j / V through the device K matvec when op_k is given."""
    torch = _torch()
    eps = _eps_dev(m)
    j = _field_dev(j, eps.numel(), "recover_fields")
    sc = _scene(m, inc)
    e = torch.empty_like(j)
    h = torch.empty_like(j) if op_k is not None else None
    with torch.cuda.device(eps.device):
        _check(lib().vie_recover_fields(None, C.byref(sc), C.c_void_p(eps.data_ptr()), C.c_void_p(j.data_ptr()),
                                        (op_k.handle if op_k is not None else None), C.c_void_p(e.data_ptr()),
                                        C.c_void_p(h.data_ptr() if h is not None else None),
                                        C.c_void_p(_stream_handle(stream, eps.device))))
    return Fields(e, h, h is not None)


@dataclass
class PostProcess:  # solver.hpp:251-256
    p_abs: object
    total_absorbed_power: float
    b1_plus: object = None
    has_b1: bool = False


def postprocess(fields: Fields, m: DielectricMap, stream=None) -> PostProcess:
    """postprocess (solver.hpp:258-284): p_abs = sigma |e|^2 / 2, total power, |b1+|."""
    torch = _torch()
    eps = _eps_dev(m)
    nv = eps.numel()
    e = _field_dev(fields.e, nv, "postprocess")
    h = _field_dev(fields.h, nv, "postprocess") if fields.has_h else None
    sc = _scene(m, None)
    p = torch.empty(nv, dtype=torch.float64, device=eps.device)
    b1 = torch.empty(nv, dtype=torch.float64, device=eps.device) if h is not None else None
    tot = C.c_double()
    with torch.cuda.device(eps.device):
        _check(lib().vie_postprocess(None, C.byref(sc), C.c_void_p(eps.data_ptr()), C.c_void_p(e.data_ptr()),
                                     C.c_void_p(h.data_ptr() if h is not None else None), C.c_void_p(p.data_ptr()),
                                     C.c_void_p(b1.data_ptr() if b1 is not None else None), C.byref(tot),
                                     C.c_void_p(_stream_handle(stream, eps.device))))
    return PostProcess(p, tot.value, b1, b1 is not None)


@dataclass
class SolveReport:  # solver.hpp:286-295
    j: object
    residual_history: list
    final_relative_residual: float
    iterations: int
    converged: bool
    wall_time_s: float
    fields: Fields
    post: PostProcess


def solve_scene(m: DielectricMap, inc: PlaneWave, op_n: EmbeddedSpectrum, op_k: "EmbeddedSpectrum | None" = None,
                cfg: GmresConfig = GmresConfig()) -> SolveReport:
    """solve_scene (solver.hpp:300-326) on the device: build_rhs, restarted GMRES on the
    JVIE system (M_eps - M_chi N / V), recover_fields, postprocess.  PWC operators."""
    import time

    torch = _torch()
    if op_n.kind != KIND_N or op_n.basis != PWC:
        raise ValueError("solve_scene: op_n must be the PWC N operator")
    if tuple(op_n.grid_dims) != tuple(int(d) for d in m.grid.dims):
        raise ValueError("apply_operator: dim mismatch")
    eps = _eps_dev(m)
    torch.cuda.synchronize(eps.device)
    t0 = time.perf_counter()
    rhs = build_rhs(m, inc)
    g = gmres(op_n, eps, 1.0 / m.grid.voxel_volume(), rhs, cfg)
    f = recover_fields(g.solution, m, inc, op_k)
    post = postprocess(f, m)
    torch.cuda.synchronize(eps.device)
    return SolveReport(g.solution, g.residual_history, g.final_relative_residual, g.iterations, g.converged,
                       time.perf_counter() - t0, f, post)
