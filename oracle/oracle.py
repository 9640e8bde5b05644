"""ctypes binding of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
The C++ source restates /root/reference/proj/include/vie (see vie_oracle.h).

Complex arrays cross the boundary as numpy complex128 (interleaved re/im,
identical to std::complex<double>).  Tensor3 data uses the reference layout
flat = i + n1*(j + n2*k); numpy arrays passed here are 1-D flat vectors or
arrays created with order='F' for (n1, n2, n3) shapes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

KIND_N, KIND_K = 0, 1
PWC, PWL = 0, 1

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_LINMAP = C.CFUNCTYPE(None, _dp, _dp, C.c_void_p)


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "vie_oracle.cpp"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_mv_npieces.argtypes = [C.c_void_p]
        L.orc_mv_piece.argtypes = [C.c_void_p, C.c_int]
        L.orc_mv_result.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_mv_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


class OracleError(ValueError):
    """Raised where the reference throws std::invalid_argument."""


def _check(rc: int):
    if rc != 0:
        raise OracleError(lib().orc_last_error().decode())


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i64(vals):
    return (C.c_int64 * len(vals))(*[int(v) for v in vals])


def set_threads(n: int):
    lib().orc_set_threads(int(n))


# ---- seeded inputs (tests/test_util.hpp:9-31) ------------------------------
def random_tensor(n1, n2, n3, seed) -> np.ndarray:
    out = np.empty(n1 * n2 * n3, np.complex128)
    _check(lib().orc_random_tensor(C.c_int64(n1), C.c_int64(n2), C.c_int64(n3), C.c_uint64(seed), _ptr(out)))
    return out


def random_matrix(rows, cols, seed) -> np.ndarray:
    """Column-major rows x cols, returned as a numpy (rows, cols) array."""
    out = np.empty(rows * cols, np.complex128)
    _check(lib().orc_random_matrix(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), _ptr(out)))
    return out.reshape((rows, cols), order="F")


def gauss_stream(seed, count) -> np.ndarray:
    out = np.empty(count, np.complex128)
    _check(lib().orc_gauss_stream(C.c_uint64(seed), C.c_int64(count), _ptr(out)))
    return out


# ---- DFT -------------------------------------------------------------------
def fft1(v, inverse=False) -> np.ndarray:
    a = _c(v).copy()
    _check(lib().orc_fft1(_ptr(a), C.c_int64(a.size), int(inverse)))
    return a


def fft3(t, dims, inverse=False) -> np.ndarray:
    a = _c(t).reshape(-1).copy()
    _check(lib().orc_fft3(_ptr(a), C.c_int64(dims[0]), C.c_int64(dims[1]), C.c_int64(dims[2]), int(inverse)))
    return a


def circulant_embed(t, dims, sign) -> np.ndarray:
    a = _c(t).reshape(-1)
    out = np.empty(8 * int(np.prod(dims)), np.complex128)
    _check(lib().orc_circulant_embed(_ptr(a), _i64(dims), (C.c_int * 3)(*sign), _ptr(out)))
    return out


def transform_factor(u, sign) -> np.ndarray:
    """u: (n, r) array -> (2n, r) embedded + DFT'd factor (operator.hpp:76-90)."""
    u = np.asarray(u, np.complex128)
    n, r = u.shape
    a = np.asfortranarray(u)
    out = np.empty(2 * n * r, np.complex128)
    _check(lib().orc_transform_factor(a.ctypes.data_as(_dp), C.c_int64(n), C.c_int64(r), int(sign), _ptr(out)))
    return out.reshape((2 * n, r), order="F")


# ---- component tables ------------------------------------------------------
def component_table(kind, basis):
    nc, nb = C.c_int(), C.c_int()
    comps = (C.c_int * (4 * 64))()
    par = (C.c_int * (3 * 64))()
    blocks = (C.c_int * (4 * 256))()
    _check(lib().orc_component_table(int(kind), int(basis), C.byref(nc), comps, par, C.byref(nb), blocks))
    c = np.array(comps[: 4 * nc.value], np.int32).reshape(-1, 4)
    p = np.array(par[: 3 * nc.value], np.int32).reshape(-1, 3)
    b = np.array(blocks[: 4 * nb.value], np.int32).reshape(-1, 4)
    return c, p, b


def ncur(basis):
    return 3 if basis == PWC else 12


# ---- Tucker forms ----------------------------------------------------------
class Form:
    """One component's Fourier-domain Tucker form (factors have 2n rows)."""

    def __init__(self, core, u1, u2, u3):
        self.core = _c(np.asarray(core).reshape(-1, order="F") if np.asarray(core).ndim == 3 else core)
        self.u = [np.asfortranarray(np.asarray(x, np.complex128)) for x in (u1, u2, u3)]
        self.ranks = [self.u[0].shape[1], self.u[1].shape[1], self.u[2].shape[1]]


def _form_arrays(forms):
    n = len(forms)
    ranks = (C.c_int64 * (3 * n))(*[r for f in forms for r in f.ranks])
    PP = _dp * n
    cores = PP(*[_ptr(f.core) for f in forms])
    u1 = PP(*[f.u[0].ctypes.data_as(_dp) for f in forms])
    u2 = PP(*[f.u[1].ctypes.data_as(_dp) for f in forms])
    u3 = PP(*[f.u[2].ctypes.data_as(_dp) for f in forms])
    return ranks, cores, u1, u2, u3


def decompress_tucker(edims, form: Form) -> np.ndarray:
    out = np.empty(int(np.prod(edims)), np.complex128)
    _check(lib().orc_decompress_tucker(_i64(edims), _i64(form.ranks), _ptr(form.core),
                                       form.u[0].ctypes.data_as(_dp), form.u[1].ctypes.data_as(_dp),
                                       form.u[2].ctypes.data_as(_dp), _ptr(out)))
    return out


def apply_operator_tucker(kind, basis, grid, forms, x) -> np.ndarray:
    x = _c(x).reshape(-1)
    y = np.empty_like(x)
    ranks, cores, u1, u2, u3 = _form_arrays(forms)
    _check(lib().orc_apply_operator_tucker(int(kind), int(basis), _i64(grid), ranks, cores, u1, u2, u3,
                                           _ptr(x), _ptr(y)))
    return y


class StagedMatvec:
    """apply_operator_tucker as the 2S + NC pieces of one matvec (orc_mv_*): the CPU
    baseline times every piece of one full matvec, spread over bench steps."""

    def __init__(self, kind, basis, grid, forms, x):
        self._keep = (forms, _form_arrays(forms))
        ranks, cores, u1, u2, u3 = self._keep[1]
        self.x = _c(x).reshape(-1)
        self.h = C.c_void_p()
        _check(lib().orc_mv_create(int(kind), int(basis), _i64(grid), ranks, cores, u1, u2, u3, _ptr(self.x),
                                   C.byref(self.h)))
        self.npieces = lib().orc_mv_npieces(self.h)

    def piece(self, i: int):
        _check(lib().orc_mv_piece(self.h, int(i)))

    def result(self) -> np.ndarray:
        y = np.empty_like(self.x)
        _check(lib().orc_mv_result(self.h, _ptr(y)))
        return y

    def close(self):
        if self.h:
            lib().orc_mv_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dense_spectrum(t, dims, sign) -> np.ndarray:
    a = _c(t).reshape(-1)
    out = np.empty(8 * int(np.prod(dims)), np.complex128)
    _check(lib().orc_dense_spectrum(_ptr(a), _i64(dims), (C.c_int * 3)(*sign), _ptr(out)))
    return out


def apply_operator_dense(kind, basis, grid, spectra, x) -> np.ndarray:
    x = _c(x).reshape(-1)
    y = np.empty_like(x)
    sp = [_c(s) for s in spectra]
    arr = (_dp * len(sp))(*[_ptr(s) for s in sp])
    _check(lib().orc_apply_operator_dense(int(kind), int(basis), _i64(grid), arr, _ptr(x), _ptr(y)))
    return y


def dense_bttb(kind, basis, dims, tensors) -> np.ndarray:
    ts = [_c(t).reshape(-1) for t in tensors]
    nv = int(np.prod(dims))
    n = ncur(basis) * nv
    out = np.empty(n * n, np.complex128)
    arr = (_dp * len(ts))(*[_ptr(t) for t in ts])
    _check(lib().orc_dense_bttb(int(kind), int(basis), _i64(dims), arr, _ptr(out)))
    return out.reshape((n, n), order="F")


def apply_system_tucker(basis, grid, forms, eps_r, inv_v, x) -> np.ndarray:
    x = _c(x).reshape(-1)
    e = _c(eps_r).reshape(-1)
    y = np.empty_like(x)
    ranks, cores, u1, u2, u3 = _form_arrays(forms)
    _check(lib().orc_apply_system_tucker(int(basis), _i64(grid), ranks, cores, u1, u2, u3, _ptr(e),
                                         C.c_double(inv_v), _ptr(x), _ptr(y)))
    return y


class GmresResult:
    def __init__(self, x, iterations, converged, final_rel, history):
        self.solution = x
        self.iterations = iterations
        self.converged = bool(converged)
        self.final_relative_residual = final_rel
        self.residual_history = history


def gmres(apply, rhs, tol=1e-5, inner=50, outer=200, x0=None, precond=None, history_cap=100000):
    """gmres (solver.hpp:34-142) with python callables for apply / precond."""
    rhs = _c(rhs).reshape(-1)
    n = rhs.size

    def wrap(fn):
        def cb(xp, yp, _ctx):
            xv = np.ctypeslib.as_array(xp, shape=(2 * n,)).view(np.complex128)
            yv = np.ctypeslib.as_array(yp, shape=(2 * n,)).view(np.complex128)
            yv[:] = fn(xv.copy())
        return _LINMAP(cb)

    ap = wrap(apply)
    pc = wrap(precond) if precond is not None else _LINMAP()
    x = np.empty(n, np.complex128)
    x0a = _c(x0).reshape(-1) if x0 is not None else None
    it, cv, hl = C.c_int(), C.c_int(), C.c_int()
    fr = C.c_double()
    hist = np.empty(history_cap, np.float64)
    _check(lib().orc_gmres(ap, None, pc, None, C.c_int64(n), _ptr(rhs),
                           _ptr(x0a) if x0a is not None else None, C.c_double(tol), int(inner), int(outer),
                           _ptr(x), C.byref(it), C.byref(cv), C.byref(fr),
                           hist.ctypes.data_as(_dp), int(history_cap), C.byref(hl)))
    return GmresResult(x, it.value, cv.value, fr.value, hist[: min(hl.value, history_cap)].copy())


def gmres_system_tucker(basis, grid, forms, eps_r, inv_v, rhs, tol=1e-5, inner=50, outer=200, x0=None,
                        history_cap=100000):
    rhs = _c(rhs).reshape(-1)
    e = _c(eps_r).reshape(-1)
    x = np.empty_like(rhs)
    x0a = _c(x0).reshape(-1) if x0 is not None else None
    ranks, cores, u1, u2, u3 = _form_arrays(forms)
    it, cv, hl = C.c_int(), C.c_int(), C.c_int()
    fr = C.c_double()
    hist = np.empty(history_cap, np.float64)
    _check(lib().orc_gmres_system_tucker(int(basis), _i64(grid), ranks, cores, u1, u2, u3, _ptr(e),
                                         C.c_double(inv_v), _ptr(rhs),
                                         _ptr(x0a) if x0a is not None else None, C.c_double(tol), int(inner),
                                         int(outer), _ptr(x), C.byref(it), C.byref(cv), C.byref(fr),
                                         hist.ctypes.data_as(_dp), int(history_cap), C.byref(hl)))
    return GmresResult(x, it.value, cv.value, fr.value, hist[: min(hl.value, history_cap)].copy())


# ---- HOSVD -----------------------------------------------------------------
def truncated_svd_values(m, tol, rule=1):
    m = np.asfortranarray(np.asarray(m, np.complex128))
    rows, cols = m.shape
    rank = C.c_int64()
    s = np.empty(min(rows, cols), np.float64)
    _check(lib().orc_truncated_svd_values(m.ctypes.data_as(_dp), C.c_int64(rows), C.c_int64(cols),
                                          C.c_double(tol), int(rule), C.byref(rank), s.ctypes.data_as(_dp)))
    return rank.value, s


def hosvd(t, dims, tol, rule=1):
    """hosvd (decomp.hpp:160-176): returns (core flat, [U1, U2, U3] (n_q, r_q))."""
    t = _c(t).reshape(-1)
    ranks = (C.c_int64 * 3)()
    _check(lib().orc_hosvd(_ptr(t), _i64(dims), C.c_double(tol), int(rule), ranks, None, None, None, None))
    r = [ranks[0], ranks[1], ranks[2]]
    core = np.empty(r[0] * r[1] * r[2], np.complex128)
    us = [np.empty(dims[q] * r[q], np.complex128) for q in range(3)]
    _check(lib().orc_hosvd(_ptr(t), _i64(dims), C.c_double(tol), int(rule), ranks, _ptr(core), _ptr(us[0]),
                           _ptr(us[1]), _ptr(us[2])))
    return core, [us[q].reshape((dims[q], r[q]), order="F") for q in range(3)]


# ---- solve_scene stages (solver.hpp:148-285) ---------------------------------
def _scene_args(scene):
    """scene: dict(dims, resolution, origin, frequency, polarization, direction, amplitude)."""
    geo = (C.c_double * 6)(*[float(v) for v in list(scene["resolution"]) + list(scene.get("origin", (0, 0, 0)))])
    pw = (C.c_double * 7)(*[float(v) for v in list(scene.get("polarization", (1, 0, 0)))
                            + list(scene.get("direction", (0, 0, 1))) + [scene.get("amplitude", 1.0)]])
    return _i64(scene["dims"]), geo, C.c_double(float(scene["frequency"])), pw


def build_rhs(scene, eps_r, quad: int = 1) -> np.ndarray:
    """build_rhs (solver.hpp:148-179): 3 n_vox complex."""
    d, geo, f, pw = _scene_args(scene)
    e = _c(eps_r).reshape(-1)
    out = np.empty(3 * e.size, np.complex128)
    _check(lib().orc_build_rhs(d, geo, f, pw, _ptr(e), C.c_int(int(quad)), _ptr(out)))
    return out


def recover_fields(scene, eps_r, j, kj=None):
    """recover_fields (solver.hpp:211-249) with K j precomputed (kj) or None: (e, h)."""
    d, geo, f, pw = _scene_args(scene)
    e_r = _c(eps_r).reshape(-1)
    jj = _c(j).reshape(-1)
    e = np.empty_like(jj)
    h = np.empty_like(jj) if kj is not None else None
    kk = _c(kj).reshape(-1) if kj is not None else None
    _check(lib().orc_recover_fields(d, geo, f, pw, _ptr(e_r), _ptr(jj), _ptr(kk) if kk is not None else None,
                                    _ptr(e), _ptr(h) if h is not None else None))
    return e, h


def postprocess(scene, eps_r, e, h=None):
    """postprocess (solver.hpp:258-284): (p_abs, total_absorbed_power, b1_plus or None)."""
    d, geo, f, _ = _scene_args(scene)
    e_r = _c(eps_r).reshape(-1)
    ee = _c(e).reshape(-1)
    p = np.empty(e_r.size, np.float64)
    b1 = np.empty(e_r.size, np.float64) if h is not None else None
    hh = _c(h).reshape(-1) if h is not None else None
    tot = C.c_double()
    _check(lib().orc_postprocess(d, geo, f, _ptr(e_r), _ptr(ee), _ptr(hh) if hh is not None else None,
                                 p.ctypes.data_as(_dp), b1.ctypes.data_as(_dp) if b1 is not None else None,
                                 C.byref(tot)))
    return p, tot.value, b1


def decompress_cp(edims, ws) -> np.ndarray:
    """decompress_cp (operator.hpp:248-261) of merged Fourier factors W_q (2n_q x R)."""
    ws = [np.asfortranarray(np.asarray(w, np.complex128)) for w in ws]
    out = np.empty(int(np.prod(edims)), np.complex128)
    _check(lib().orc_decompress_cp(_i64(edims), C.c_int64(ws[0].shape[1]), ws[0].ctypes.data_as(_dp),
                                   ws[1].ctypes.data_as(_dp), ws[2].ctypes.data_as(_dp), _ptr(out)))
    return out


class CpAls:
    def __init__(self, factors, trace, converged, ill_posed):
        self.factors, self.trace, self.converged, self.ill_posed = factors, trace, converged, ill_posed


def cp_als(t, dims, r, max_iters=100, stall_tol=1e-12, seed=0x5EED) -> CpAls:
    """cp_als (decomp.hpp:237-298): factors (dims[q], r), per-sweep relative error trace."""
    t = _c(t).reshape(-1)
    fs = [np.empty(dims[q] * r, np.complex128) for q in range(3)]
    cap = max(int(max_iters), 1) + 1
    tr = np.empty(cap)
    nt = C.c_int()
    flags = (C.c_int * 2)()
    _check(lib().orc_cp_als(_ptr(t), _i64(dims), C.c_int64(r), int(max_iters), C.c_double(stall_tol),
                            C.c_uint64(seed), _ptr(fs[0]), _ptr(fs[1]), _ptr(fs[2]),
                            tr.ctypes.data_as(_dp), cap, C.byref(nt), flags))
    return CpAls([fs[q].reshape((dims[q], r), order="F") for q in range(3)], tr[:nt.value].copy(),
                 bool(flags[0]), bool(flags[1]))


class TuckerCp:
    def __init__(self, factors, rank, hosvd_err, core_err, achieved, trace):
        self.factors, self.rank = factors, rank
        self.hosvd_relative_error, self.core_cp_relative_error = hosvd_err, core_err
        self.achieved_relative_error, self.trace = achieved, trace


def tucker_cp(t, dims, tol, cp_iters=1000, rule=1, cp_rank=-1, stall_tol=0.0) -> TuckerCp:
    """tucker_cp (decomp.hpp:336-373): merged factors W_q = U_q V_q (dims[q], rank)."""
    t = _c(t).reshape(-1)
    rk = C.c_int64()
    nt = C.c_int()
    errs = (C.c_double * 3)()
    args = (_ptr(t), _i64(dims), C.c_double(tol), int(cp_iters), int(rule), C.c_int64(cp_rank), C.c_double(stall_tol))
    _check(lib().orc_tucker_cp(*args, C.byref(rk), None, None, None, errs, None, 0, C.byref(nt)))
    r = rk.value
    ws = [np.empty(dims[q] * r, np.complex128) for q in range(3)]
    cap = int(cp_iters) + 1
    tr = np.empty(cap)
    _check(lib().orc_tucker_cp(*args, C.byref(rk), _ptr(ws[0]), _ptr(ws[1]), _ptr(ws[2]), errs,
                               tr.ctypes.data_as(_dp), cap, C.byref(nt)))
    return TuckerCp([ws[q].reshape((dims[q], r), order="F") for q in range(3)], r, errs[0], errs[1], errs[2],
                    tr[:nt.value].copy())


# ---- Green's-tensor assembly (assembly.hpp, kernels.hpp, quadrature.hpp) ---------
OP_N, OP_K, OP_G, OP_NREM = 0, 1, 2, 3


def _quad5(quad):
    if quad is None:
        return None
    return (C.c_int * 5)(*[int(v) for v in quad])


def assemble(dims, res, k0, op, q, qp, quad=None) -> np.ndarray:
    """assemble_defining_tensor (assembly.hpp:159-233), PWC; flat reference layout."""
    out = np.empty(int(np.prod(dims)), np.complex128)
    _check(lib().orc_assemble(_i64(dims), (C.c_double * 3)(*[float(r) for r in res]), C.c_double(k0), int(op),
                              int(q), int(qp), _quad5(quad), _ptr(out)))
    return out


def self_static_term(delta, quad=None):
    """self_static_term (assembly.hpp:127-150): (dyad diagonal, gram, error, converged)."""
    dg = (C.c_double * 3)()
    gram, err, conv = C.c_double(), C.c_double(), C.c_int()
    _check(lib().orc_self_static_term((C.c_double * 3)(*delta), _quad5(quad), dg, C.byref(gram), C.byref(err),
                                      C.byref(conv)))
    return np.array(dg[:]), gram.value, err.value, bool(conv.value)


def correlation_entry(op, k, q, qp, d, delta, points, duffy=False) -> complex:
    out = (C.c_double * 2)()
    _check(lib().orc_correlation_entry(int(op), C.c_double(k), int(q), int(qp), (C.c_double * 3)(*d),
                                       (C.c_double * 3)(*delta), int(points), int(bool(duffy)), out))
    return complex(out[0], out[1])


def kernel_eval(op, k, q, qp, r) -> complex:
    out = (C.c_double * 2)()
    _check(lib().orc_kernel_eval(int(op), C.c_double(k), int(q), int(qp), (C.c_double * 3)(*r), out))
    return complex(out[0], out[1])


def radial(R, k, dynamic=False):
    out = (C.c_double * 6)()
    _check(lib().orc_radial(C.c_double(R), C.c_double(k), int(bool(dynamic)), out))
    return tuple(complex(out[2 * i], out[2 * i + 1]) for i in range(3))


def brute_pair_integral(op, k, q, qp, d, delta, p) -> complex:
    out = (C.c_double * 2)()
    _check(lib().orc_brute_pair_integral(int(op), C.c_double(k), int(q), int(qp), (C.c_double * 3)(*d),
                                         (C.c_double * 3)(*delta), int(p), out))
    return complex(out[0], out[1])
