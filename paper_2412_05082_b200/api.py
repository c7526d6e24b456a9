"""Thin Python binding over the C ABI (include/c0ip.h): torch tensors in, device pointers out.

Every computation runs in the CUDA library; this module only marshals arguments.
PyTorch provides device memory and the current stream.
"""
import ctypes as C

import numpy as np
import torch

from . import _lib as L

_DT = {torch.float64: L.F64, torch.float32: L.F32}
SMOOTHERS = {"avs_atomic": L.AVS_ATOMIC, "avs": L.AVS_DETERMINISTIC, "avs_det": L.AVS_DETERMINISTIC,
             "avs_colored": L.AVS_COLORED, "mvs": L.MVS}


def _ptr(t):
    if not t.is_cuda:
        raise ValueError("tensor must be on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}") from None


def _check(ref, n, *ts):
    """Every tensor: same dtype and device as `ref`, contiguous, n elements (argument marshalling
    only; the library cannot see tensor lengths and would read/write out of bounds)."""
    for t in (ref,) + ts:
        if t is None:
            continue
        if t.dtype != ref.dtype or t.device != ref.device:
            raise ValueError(f"tensor dtype/device {t.dtype}/{t.device} != {ref.dtype}/{ref.device}")
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if t.numel() != n:
            raise ValueError(f"tensor has {t.numel()} elements, expected {n}")


class MG:
    """c0ip_mg_config: smoother, steps, omega, symmetric, cycle dtype (torch.float64/float32)."""

    def __init__(self, smoother="avs", steps=2, omega=0.25, symmetric=True, cycle_dtype=torch.float64):
        self.c = L.MgConfig(SMOOTHERS[smoother] if isinstance(smoother, str) else int(smoother), int(steps),
                            float(omega), int(bool(symmetric)), _DT[cycle_dtype])


class Context:
    def __init__(self, dim, degree, finest_level, cells_override=0, penalty_scale=1.0, device=0, nodes=None,
                 sipg=False):
        """nodes: optional per-axis cell boundaries of the finest level (graded mesh, c0ip_create_graded);
        sipg: the Poisson SIPG comparison workload (c0ip_create_sipg)."""
        self._lib = L.load()
        cfg = L.Config(int(dim), int(degree), int(finest_level), int(cells_override), float(penalty_scale),
                       int(device))
        h = C.c_void_p()
        if sipg:
            L.check(self._lib.c0ip_create_sipg(C.byref(cfg), C.byref(h)))
        elif nodes is None:
            L.check(self._lib.c0ip_create(C.byref(cfg), C.byref(h)))
        else:
            self._nodes = [None if x is None else np.ascontiguousarray(x, dtype=np.float64) for x in nodes]
            ptrs = (C.c_void_p * 3)(*[None if x is None else x.ctypes.data for x in self._nodes + [None] * (3 - len(self._nodes))])
            L.check(self._lib.c0ip_create_graded(C.byref(cfg), ptrs, C.byref(h)))
        self.h = h
        self.dim, self.degree = int(dim), int(degree)
        self.sipg = bool(sipg)
        self.finest_level = int(finest_level)
        self.device = torch.device("cuda", int(device))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self._lib.c0ip_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ host-side maps
    def set_path(self, generic):
        L.check(self._lib.c0ip_set_path(self.h, L.PATH_GENERIC if generic else L.PATH_AUTO))

    def set_local_solver(self, exact):
        """FDM surrogate (default, Eq. localsolverbila) or exact patch matrices A_v (Table 1)."""
        L.check(self._lib.c0ip_set_local_solver(self.h, L.LOCAL_EXACT if exact else L.LOCAL_FDM))

    def level_info(self, level):
        nd, n1, nc, npch = (C.c_int64() for _ in range(4))
        ncol = C.c_int32()
        L.check(self._lib.c0ip_level_info(self.h, level, C.byref(nd), C.byref(n1), C.byref(nc), C.byref(npch),
                                          C.byref(ncol)))
        return dict(n_dofs=nd.value, n_1d=n1.value, cells=nc.value, n_patches=npch.value, n_colors=ncol.value)

    def patch_dofs(self, level, patch):
        out = np.empty((2 * self.degree + (2 if self.sipg else -1)) ** self.dim, dtype=np.int64)
        L.check(self._lib.c0ip_patch_dofs(self.h, level, patch, out.ctypes.data_as(C.c_void_p)))
        return out

    def color_patches(self, level, color):
        cnt = C.c_int64()
        L.check(self._lib.c0ip_color_patches(self.h, level, color, None, 0, C.byref(cnt)))
        out = np.empty(cnt.value, dtype=np.int64)
        L.check(self._lib.c0ip_color_patches(self.h, level, color, out.ctypes.data_as(C.c_void_p), cnt.value,
                                             C.byref(cnt)))
        return out

    def fdm(self, level, variant):
        np_ = 2 * self.degree + (2 if self.sipg else -1)
        S = np.empty((np_, np_)); lam = np.empty(np_)
        L.check(self._lib.c0ip_get_fdm(self.h, level, variant, S.ctypes.data_as(C.c_void_p),
                                       lam.ctypes.data_as(C.c_void_p)))
        return S, lam

    def matrices_1d(self, level):
        n = self.level_info(level)["n_1d"]
        M, Lm, B = (np.empty((n, n)) for _ in range(3))
        L.check(self._lib.c0ip_get_matrices_1d(self.h, level, *(X.ctypes.data_as(C.c_void_p) for X in (M, Lm, B))))
        return M, Lm, B

    def launch_count(self):
        c = C.c_int64()
        L.check(self._lib.c0ip_launch_count(self.h, C.byref(c)))
        return c.value

    # ------------------------------------------------------------------ device ops
    def n_dofs(self, level):
        return self.level_info(level)["n_dofs"]

    def _n(self, level):
        return self.n_dofs(level)              # the ABI rejects a bad level (C0IP_ERR_ARG)

    def rhs(self, level):
        b = torch.empty(self.n_dofs(level), dtype=torch.float64, device=self.device)
        L.check(self._lib.c0ip_rhs(self.h, level, _ptr(b), _stream()))
        return b

    def apply(self, level, x, y=None):
        y = torch.empty_like(x) if y is None else y
        _check(x, self._n(level), y)
        L.check(self._lib.c0ip_apply(self.h, level, _dtype(x), _ptr(x), _ptr(y), _stream()))
        return y

    def residual(self, level, b, x, r=None):
        r = torch.empty_like(x) if r is None else r
        _check(x, self._n(level), b, r)
        L.check(self._lib.c0ip_residual(self.h, level, _dtype(x), _ptr(b), _ptr(x), _ptr(r), _stream()))
        return r

    def smooth(self, level, smoother, steps, omega, b, x, reverse=False):
        sm = SMOOTHERS[smoother] if isinstance(smoother, str) else int(smoother)
        _check(x, self._n(level), b)
        L.check(self._lib.c0ip_smooth(self.h, level, _dtype(x), sm, int(steps), float(omega), int(bool(reverse)),
                                      _ptr(b), _ptr(x), _stream()))
        return x

    def restrict(self, fine_level, fine, coarse=None):
        if coarse is None:
            coarse = torch.empty(self.n_dofs(fine_level - 1), dtype=fine.dtype, device=fine.device)
        if fine_level < 2:
            raise ValueError("restrict needs fine_level >= 2")
        _check(fine, self._n(fine_level))
        _check(coarse, self._n(fine_level - 1))
        if coarse.dtype != fine.dtype or coarse.device != fine.device:
            raise ValueError("coarse and fine tensors differ in dtype/device")
        L.check(self._lib.c0ip_restrict(self.h, fine_level, _dtype(fine), _ptr(fine), _ptr(coarse), _stream()))
        return coarse

    def prolongate_add(self, fine_level, coarse, fine):
        if fine_level < 2:
            raise ValueError("prolongate_add needs fine_level >= 2")
        _check(fine, self._n(fine_level))
        _check(coarse, self._n(fine_level - 1))
        if coarse.dtype != fine.dtype or coarse.device != fine.device:
            raise ValueError("coarse and fine tensors differ in dtype/device")
        L.check(self._lib.c0ip_prolongate_add(self.h, fine_level, _dtype(fine), _ptr(coarse), _ptr(fine),
                                              _stream()))
        return fine

    def vcycle(self, mg, r, z=None):
        z = torch.empty_like(r) if z is None else z
        if r.dtype != torch.float64:
            raise ValueError("vcycle takes FP64 vectors (the cycle dtype is set in MG)")
        _check(r, self._n(self.finest_level), z)
        L.check(self._lib.c0ip_vcycle(self.h, C.byref(mg.c), _ptr(r), _ptr(z), _stream()))
        return z

    def pcg(self, mg, b, x=None, rtol=1e-8, max_iter=200):
        x = torch.zeros_like(b) if x is None else x
        if b.dtype != torch.float64:
            raise ValueError("pcg takes FP64 vectors")
        _check(b, self._n(self.finest_level), x)
        rep = L.Report()
        hist = np.zeros(max_iter + 1)
        L.check(self._lib.c0ip_pcg(self.h, C.byref(mg.c), _ptr(b), _ptr(x), float(rtol), int(max_iter),
                                   C.byref(rep), hist.ctypes.data_as(C.c_void_p), _stream()))
        report = dict(iterations=rep.iterations, converged=bool(rep.converged), r0=rep.r0, rn=rep.rn, nu=rep.nu,
                      seconds=rep.seconds)
        return x, report, hist[: rep.iterations + 1]

    def gmres(self, mg, b, x=None, rtol=1e-8, max_iter=200, restart=50):
        """Flexible right-preconditioned GMRES(restart) in FP64 around the V-cycle (c0ip_gmres)."""
        x = torch.zeros_like(b) if x is None else x
        if b.dtype != torch.float64:
            raise ValueError("gmres takes FP64 vectors")
        _check(b, self._n(self.finest_level), x)
        rep = L.Report()
        hist = np.zeros(max_iter + 1)
        L.check(self._lib.c0ip_gmres(self.h, C.byref(mg.c), _ptr(b), _ptr(x), float(rtol), int(max_iter),
                                     int(restart), C.byref(rep), hist.ctypes.data_as(C.c_void_p), _stream()))
        report = dict(iterations=rep.iterations, converged=bool(rep.converged), r0=rep.r0, rn=rep.rn, nu=rep.nu,
                      seconds=rep.seconds)
        return x, report, hist[: rep.iterations + 1]

    # ------------------------------------------------------------------ slab (multi-GPU) calls
    def slab_ghosts(self):
        ga, gp = C.c_int32(), C.c_int32()
        L.check(self._lib.c0ip_slab_ghosts(self.h, C.byref(ga), C.byref(gp)))
        return ga.value, gp.value

    def _slab_n(self, level, lrows):
        n1 = self.level_info(level)["n_1d"]
        return int(lrows) * n1 ** (self.dim - 1)

    def slab_avs_step(self, level, omega, row0, lrows, out_lo, out_hi, b_ext, x_ext, r_ext):
        _check(x_ext, self._slab_n(level, lrows), b_ext, r_ext)
        L.check(self._lib.c0ip_slab_avs_step(self.h, level, _dtype(x_ext), float(omega), int(row0), int(lrows),
                                             int(out_lo), int(out_hi), _ptr(b_ext), _ptr(x_ext), _ptr(r_ext),
                                             _stream()))
        return x_ext

    def slab_apply(self, level, row0, lrows, out_lo, out_hi, x_ext, y_ext, b_ext=None):
        _check(x_ext, self._slab_n(level, lrows), y_ext, b_ext)
        L.check(self._lib.c0ip_slab_apply(self.h, level, _dtype(x_ext), int(row0), int(lrows), int(out_lo),
                                          int(out_hi), _ptr(b_ext) if b_ext is not None else None, _ptr(x_ext),
                                          _ptr(y_ext), _stream()))
        return y_ext

    def slab_fdm(self, level, omega, row0, lrows, out_lo, out_hi, r_ext, x_ext):
        _check(x_ext, self._slab_n(level, lrows), r_ext)
        L.check(self._lib.c0ip_slab_fdm(self.h, level, _dtype(x_ext), float(omega), int(row0), int(lrows), int(out_lo),
                                        int(out_hi), _ptr(r_ext), _ptr(x_ext), _stream()))
        return x_ext

    def slab_mvs_color(self, level, omega, color, row0, lrows, out_lo, out_hi, b_ext, x_ext, r_ext):
        _check(x_ext, self._slab_n(level, lrows), b_ext, r_ext)
        L.check(self._lib.c0ip_slab_mvs_color(self.h, level, _dtype(x_ext), float(omega), int(color), int(row0),
                                              int(lrows), int(out_lo), int(out_hi), _ptr(b_ext), _ptr(x_ext),
                                              _ptr(r_ext), _stream()))
        return x_ext

    def slab_restrict(self, fine_level, f_row0, f_lrows, fine_ext, c_row0, c_lrows, c_out_lo, c_out_hi, coarse_ext):
        _check(fine_ext, self._slab_n(fine_level, f_lrows))
        _check(coarse_ext, self._slab_n(fine_level - 1, c_lrows))
        L.check(self._lib.c0ip_slab_restrict(self.h, fine_level, _dtype(fine_ext), int(f_row0), int(f_lrows),
                                             _ptr(fine_ext), int(c_row0), int(c_lrows), int(c_out_lo), int(c_out_hi),
                                             _ptr(coarse_ext), _stream()))
        return coarse_ext

    def slab_prolongate_add(self, fine_level, c_row0, c_lrows, coarse_ext, f_row0, f_lrows, f_out_lo, f_out_hi,
                            fine_ext):
        _check(fine_ext, self._slab_n(fine_level, f_lrows))
        _check(coarse_ext, self._slab_n(fine_level - 1, c_lrows))
        L.check(self._lib.c0ip_slab_prolongate_add(self.h, fine_level, _dtype(fine_ext), int(c_row0), int(c_lrows),
                                                   _ptr(coarse_ext), int(f_row0), int(f_lrows), int(f_out_lo),
                                                   int(f_out_hi), _ptr(fine_ext), _stream()))
        return fine_ext

    def slab_transfer_rows(self, fine_level, c_out_lo, c_out_hi, f_out_lo, f_out_hi):
        fn, cn = (C.c_int64 * 2)(), (C.c_int64 * 2)()
        L.check(self._lib.c0ip_slab_transfer_rows(self.h, fine_level, int(c_out_lo), int(c_out_hi), int(f_out_lo),
                                                  int(f_out_hi), fn, cn))
        return (fn[0], fn[1]), (cn[0], cn[1])

    def vcycle_level(self, mg, level, r, z=None):
        z = torch.empty_like(r) if z is None else z
        if r.dtype != torch.float64:
            raise ValueError("vcycle_level takes FP64 vectors")
        _check(r, self._n(level), z)
        L.check(self._lib.c0ip_vcycle_level(self.h, C.byref(mg.c), int(level), _ptr(r), _ptr(z), _stream()))
        return z

    def axpby(self, alpha, x, beta, y):
        """y = alpha x + beta y (library kernel; x, y same dtype/device/length)."""
        _check(x, x.numel(), y)
        L.check(self._lib.c0ip_vec_axpby(self.h, _dtype(x), x.numel(), float(alpha), _ptr(x), float(beta), _ptr(y),
                                         _stream()))
        return y

    def dots(self, x0, y0, x1=None, y1=None):
        """[<x0,y0>] or [<x0,y0>, <x1,y1>] in FP64 (library kernels, synchronises)."""
        if x0.dtype != torch.float64:
            raise ValueError("dots takes FP64 vectors")
        _check(x0, x0.numel(), y0, x1, y1)
        nd = 1 if x1 is None else 2
        out = np.zeros(nd)
        L.check(self._lib.c0ip_vec_dots(self.h, x0.numel(), nd, _ptr(x0), _ptr(y0), _ptr(x1) if x1 is not None else None,
                                        _ptr(y1) if y1 is not None else None, out.ctypes.data_as(C.c_void_p),
                                        _stream()))
        return out
