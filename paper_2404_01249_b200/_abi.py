"""ctypes mirror of include/difform_gpu.h and a generic call table.

The same marshalling drives the product library (libdifform_cuda.so, entry
points ``dfm_*`` taking a ``dfm_ctx*`` first) and, in tests only, the CPU
checkers (``orc_*`` / ``dfmref_*`` without a context), because the C-ABI keeps
one argument convention for all of them.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np

DFM_OK, DFM_E_INVALID, DFM_E_NUMERICAL, DFM_E_CUDA = 0, 1, 2, 3
PREC_F32, PREC_F64 = 0, 1
HOST_F32, HOST_F64 = 0, 1
LOSS_SSD, LOSS_LNCC, LOSS_DICE = 0, 1, 2
MODE_DIRECT, MODE_SVF = 0, 1
INIT_NONE, INIT_AFFINE, INIT_FIELD = 0, 1, 2
NUM_KCLASS = 7


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference (status DFM_E_INVALID)."""


class NumericalError(RuntimeError):
    """std::runtime_error in the reference (status DFM_E_NUMERICAL)."""


class DeviceError(RuntimeError):
    """CUDA failure (status DFM_E_CUDA); no reference counterpart."""


class dfm_grid(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("dims", C.c_int64 * 3),
                ("spacing", C.c_double * 3), ("origin", C.c_double * 3)]


class dfm_config(C.Structure):
    _fields_ = [("loss", C.c_int32), ("lncc_radius", C.c_int32), ("eta", C.c_double),
                ("sigma_grad", C.c_double), ("sigma_warp", C.c_double),
                ("use_jac", C.c_int32), ("mode", C.c_int32), ("svf_M", C.c_int32),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps_adam", C.c_double),
                ("step_cap", C.c_double), ("conv_window", C.c_int32),
                ("conv_tol", C.c_double), ("seed", C.c_uint64)]


class dfm_iter_record(C.Structure):
    _fields_ = [("scale_index", C.c_int32), ("scale", C.c_double), ("iter", C.c_int32),
                ("global_iter", C.c_int64), ("loss", C.c_double),
                ("max_step", C.c_double), ("wall_ms", C.c_double)]


class dfm_init(C.Structure):
    _fields_ = [("kind", C.c_int32), ("affine_ndim", C.c_int32), ("A", C.c_double * 9),
                ("t", C.c_double * 3), ("field_grid", dfm_grid),
                ("field", C.POINTER(C.c_double))]


class dfm_runlog(C.Structure):
    _fields_ = [("n_records", C.c_int64), ("n_total", C.c_int64),
                ("final_loss", C.c_double), ("final_singularity_fraction", C.c_double),
                ("total_ms", C.c_double)]


class dfm_affine_result(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("A", C.c_double * 9), ("t", C.c_double * 3),
                ("loss", C.c_double), ("diverged", C.c_int32), ("iterations", C.c_int64)]


class dfm_region_overlap(C.Structure):
    _fields_ = [("label", C.c_int32), ("has_to", C.c_int32), ("has_fn", C.c_int32),
                ("has_fp", C.c_int32), ("fixed_count", C.c_int64), ("warped_count", C.c_int64),
                ("intersection", C.c_int64), ("to", C.c_double), ("mo", C.c_double),
                ("fn", C.c_double), ("fp", C.c_double), ("vs", C.c_double)]


class dfm_overlap_summary(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("to_mean", "mo_mean", "fn_mean", "fp_mean", "vs_mean",
                                          "to_klein", "mo_klein", "fn_klein", "fp_klein",
                                          "vs_klein")] + [("n_regions", C.c_int64)]


class dfm_sweep_pair(C.Structure):
    _fields_ = [("grid", C.c_void_p), ("fixed", C.POINTER(C.c_double)),
                ("moving", C.POINTER(C.c_double)), ("fixed_labels", C.POINTER(C.c_int32)),
                ("moving_labels", C.POINTER(C.c_int32))]


class dfm_sweep_row(C.Structure):
    _fields_ = [("eta", C.c_double), ("sigma_warp", C.c_double), ("sigma_grad", C.c_double),
                ("metric_mean", C.c_double), ("metric_sd", C.c_double), ("wall_ms", C.c_double),
                ("failed", C.c_int32), ("computed", C.c_int32), ("error", C.c_char * 256)]


SWEEP_LOSS, SWEEP_OVERLAP = 0, 1
MET_OTHER, MET_FLOAT, MET_SHORT = -1, 0, 1


class dfm_mhd_info(C.Structure):
    _fields_ = [("grid", dfm_grid), ("element_type", C.c_int32), ("channels", C.c_int32),
                ("element_type_name", C.c_char * 32), ("raw_path", C.c_char * 1024)]


# --------------------------------------------------------------------------
# host-side value types (difform::GridMeta / RegistrationConfig / ...)

@dataclass(frozen=True)
class GridMeta:
    """difform::GridMeta (core.hpp:13-23). dims are (x, y, z), x fastest."""
    ndim: int
    dims: tuple
    spacing: tuple = (1.0, 1.0, 1.0)
    origin: tuple = (0.0, 0.0, 0.0)

    @staticmethod
    def make_3d(nx, ny, nz, sx=1.0, sy=1.0, sz=1.0) -> "GridMeta":
        return GridMeta(3, (int(nx), int(ny), int(nz)), (sx, sy, sz))

    @staticmethod
    def make_2d(nx, ny, sx=1.0, sy=1.0) -> "GridMeta":
        return GridMeta(2, (int(nx), int(ny), 1), (sx, sy, 1.0))

    @property
    def voxel_count(self) -> int:
        return int(self.dims[0] * self.dims[1] * self.dims[2])

    @property
    def shape(self) -> tuple:
        """numpy shape of an image on this grid (z, y, x)."""
        return (self.dims[2], self.dims[1], self.dims[0])

    @property
    def field_shape(self) -> tuple:
        return self.shape + (self.ndim,)

    def c(self) -> dfm_grid:
        g = dfm_grid()
        g.ndim = self.ndim
        for a in range(3):
            g.dims[a] = int(self.dims[a])
            g.spacing[a] = float(self.spacing[a])
            g.origin[a] = float(self.origin[a])
        return g

    @staticmethod
    def from_c(g: dfm_grid) -> "GridMeta":
        return GridMeta(int(g.ndim), tuple(int(v) for v in g.dims),
                        tuple(float(v) for v in g.spacing), tuple(float(v) for v in g.origin))


@dataclass
class RegistrationConfig:
    """difform::RegistrationConfig with its defaults (pipeline.hpp:25-41)."""
    loss: int = LOSS_SSD
    lncc_radius: int = 2
    eta: float = 0.5
    sigma_grad: float = 1.0
    sigma_warp: float = 0.5
    use_jac: bool = False
    mode: int = MODE_DIRECT
    svf_M: int = 6
    beta1: float = 0.9
    beta2: float = 0.999
    eps_adam: float = 1e-8
    step_cap: float = 0.5
    conv_window: int = 10
    conv_tol: float = 1e-5
    seed: int = 0

    def c(self) -> dfm_config:
        c = dfm_config()
        for name, _ in dfm_config._fields_:
            setattr(c, name, int(getattr(self, name)) if name in
                    ("loss", "lncc_radius", "use_jac", "mode", "svf_M", "conv_window", "seed")
                    else float(getattr(self, name)))
        return c


@dataclass
class PyramidSchedule:
    """difform::PyramidSchedule (pipeline.hpp:14-19)."""
    scales: Sequence[float] = (4.0, 2.0, 1.0)
    iterations: Sequence[int] = (50, 50, 50)


@dataclass
class AffineTransform:
    """difform::AffineTransform (affine.hpp:12-16), voxel units, row-major A."""
    ndim: int = 3
    A: Sequence[float] = (1, 0, 0, 0, 1, 0, 0, 0, 1)
    t: Sequence[float] = (0, 0, 0)


@dataclass
class IterationRecord:
    scale_index: int
    scale: float
    iter: int
    global_iter: int
    loss: float
    max_step: float
    wall_ms: float


@dataclass
class RunLog:
    iterations: list = dc_field(default_factory=list)
    final_loss: float = 0.0
    final_singularity_fraction: float = 0.0
    total_ms: float = 0.0


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ipptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _affine_A(A, ndim) -> np.ndarray:
    """row-major ndim x ndim matrix packed into the 9-slot C array"""
    a = np.asarray(A, dtype=np.float64).reshape(ndim, ndim)
    out = np.zeros(9)
    out[:ndim * ndim] = a.ravel()
    return out


def _vec3(v) -> np.ndarray:
    out = np.zeros(3)
    v = np.asarray(v, dtype=np.float64).ravel()
    out[:len(v)] = v
    return out


def as_f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and out.shape != tuple(shape):
        out = out.reshape(shape)
    return out


# prototypes, without the leading context argument
_D = C.POINTER(C.c_double)
_G = C.POINTER(dfm_grid)
_I = C.POINTER(C.c_int32)
PROTOS = {
    "downsample_image": [_G, _D, _D, _G, _D],
    "sample_linear_points": [_G, _D, C.c_int64, _D, _D, _D],
    "warp_image": [_G, _D, _D, _D],
    "warp_labels": [_G, _I, _D, _I],
    "compose": [_G, _D, _D, _D],
    "exp_map": [_G, _D, C.c_int, _D],
    "overlap_report": [_G, _I, _G, _I, C.POINTER(dfm_overlap_summary),
                       C.POINTER(dfm_region_overlap), C.c_int64],
    "landmark_error": [_G, _G, _G, _D, C.c_int64, _D, _D, _D, _D, _D],
    "affine_to_field": [_G, _D, _D, _D],
    "affine_param_gradient": [_G, _D, _D, C.c_int, _D, _D, _D, C.c_int, _D, _D, _D],
    "affine_register": [_G, _D, _D, C.c_int, _D, _I, C.c_int32, C.c_double, C.c_int,
                        C.POINTER(dfm_affine_result)],
    "svf_pullback": [_G, _D, _D, C.c_int, _D],
    "jacobian_det": [_G, _D, _D],
    "gaussian_smooth": [_G, _D, _D, _D],
    "gaussian_smooth_field": [_G, _D, _D, _D],
    "upsample_field": [_G, _D, _G, _D],
    "resample_field_linear": [_G, _D, _G, _D],
    "resample_displacement": [_G, _D, _G, _D],
    "ssd_eval": [_G, _D, _G, _D, _D, _D, _D],
    "lncc_eval": [_G, _D, _G, _D, _D, C.c_int, _D, _D],
    "dice_eval": [_G, _D, _G, _D, _D, _D, _D],
    "adam_step": [_G, _D, _D, C.POINTER(C.c_int64), C.c_double, C.c_double, C.c_double, _D, _D],
    "upsample_state": [_G, _D, _D, _G, _D, _D],
    "eulerian_direction": [_G, _D, _D, C.c_int, _D],
    "apply_update": [_G, _D, _D, C.c_double, C.c_double, C.c_double, _D],
    "singularity_fraction": [_G, _D, _D],
}


class CallTable:
    """Binds ``<prefix><name>`` symbols of a C-ABI library.

    ``ctx`` (a c_void_p) is passed first when given, so the same table serves
    the CUDA library (ctx) and the CPU checkers (no ctx).
    """

    def __init__(self, lib: C.CDLL, prefix: str, ctx=None, err_fn: str = "dfm_last_error"):
        self.lib = lib
        self.prefix = prefix
        self.ctx = ctx
        self._err = getattr(lib, err_fn)
        self._err.restype = C.c_size_t
        self._err.argtypes = [C.c_char_p, C.c_size_t]
        self._fns = {}

    def has(self, name: str) -> bool:
        return hasattr(self.lib, self.prefix + name)

    def fn(self, name: str):
        f = self._fns.get(name)
        if f is None:
            f = getattr(self.lib, self.prefix + name)
            argtypes = list(PROTOS.get(name, []))
            if self.ctx is not None:
                argtypes = [C.c_void_p] + argtypes
            if name in PROTOS:
                f.argtypes = argtypes
            f.restype = C.c_int
            self._fns[name] = f
        return f

    def last_error(self) -> str:
        buf = C.create_string_buffer(1024)
        self._err(buf, 1024)
        return buf.value.decode(errors="replace")

    def check(self, rc: int, what: str):
        if rc == DFM_OK:
            return
        msg = f"{what}: {self.last_error()}"
        if rc == DFM_E_INVALID:
            raise InvalidArgument(msg)
        if rc == DFM_E_NUMERICAL:
            raise NumericalError(msg)
        raise DeviceError(msg)

    def call(self, name: str, *args):
        f = self.fn(name)
        rc = f(self.ctx, *args) if self.ctx is not None else f(*args)
        self.check(rc, name)


def _sigma3(sigma) -> np.ndarray:
    if np.isscalar(sigma):
        return np.array([sigma, sigma, sigma], dtype=np.float64)
    s = np.zeros(3)
    s[:len(sigma)] = sigma
    return s


class HostAPI:
    """numpy-level mirror of the difform:: operator API over one CallTable.

    Images are arrays shaped grid.shape (z, y, x); fields grid.field_shape
    (z, y, x, ndim) — i.e. the reference's x-fastest AoS memory layout.
    """

    def __init__(self, table: CallTable):
        self.t = table

    # -- core
    def downsample_image(self, g: GridMeta, img, factor):
        f = _sigma3(factor)
        f[g.ndim:] = 1.0
        img = as_f64(img, g.shape)
        og = dfm_grid()
        out = np.empty(img.size)  # upper bound
        self.t.call("downsample_image", C.byref(g.c()), _dptr(img), _dptr(f), C.byref(og),
                    _dptr(out))
        ng = GridMeta.from_c(og)
        return ng, out[:ng.voxel_count].reshape(ng.shape).copy()

    # -- interp
    def sample_linear_points(self, g: GridMeta, img, points):
        img = as_f64(img, g.shape)
        pts = as_f64(points).reshape(-1, 3)
        vals = np.empty(len(pts))
        grads = np.empty((len(pts), 3))
        self.t.call("sample_linear_points", C.byref(g.c()), _dptr(img), len(pts), _dptr(pts),
                    _dptr(vals), _dptr(grads))
        return vals, grads

    def warp_image(self, g, img, phi):
        img, phi = as_f64(img, g.shape), as_f64(phi, g.field_shape)
        out = np.empty(g.shape)
        self.t.call("warp_image", C.byref(g.c()), _dptr(img), _dptr(phi), _dptr(out))
        return out

    def warp_labels(self, g, labels, phi):
        lab = np.ascontiguousarray(labels, dtype=np.int32).reshape(g.shape)
        phi = as_f64(phi, g.field_shape)
        out = np.empty(g.shape, dtype=np.int32)
        self.t.call("warp_labels", C.byref(g.c()), _ipptr(lab), _dptr(phi), _ipptr(out))
        return out

    def compose(self, g, phi, psi):
        phi, psi = as_f64(phi, g.field_shape), as_f64(psi, g.field_shape)
        out = np.empty(g.field_shape)
        self.t.call("compose", C.byref(g.c()), _dptr(phi), _dptr(psi), _dptr(out))
        return out

    def affine_to_field(self, g, A, t):
        """affine_to_field (affine.hpp:29-30): u(x) = (A - I) x + t."""
        out = np.empty(g.field_shape)
        self.t.call("affine_to_field", C.byref(g.c()), _dptr(_affine_A(A, g.ndim)),
                    _dptr(_vec3(t)), _dptr(out))
        return out

    def affine_param_gradient(self, g, fixed, moving, loss, A, t, scale_to_full=(1, 1, 1),
                              lncc_radius=2):
        """affine_param_gradient (affine.hpp:43-46) -> (value, dA (d x d), dt (d))."""
        f, m = as_f64(fixed, g.shape), as_f64(moving, g.shape)
        val = C.c_double()
        dA = np.zeros(9)
        dt = np.zeros(3)
        self.t.call("affine_param_gradient", C.byref(g.c()), _dptr(f), _dptr(m), int(loss),
                    _dptr(_affine_A(A, g.ndim)), _dptr(_vec3(t)), _dptr(_vec3(scale_to_full)),
                    int(lncc_radius), C.byref(val), _dptr(dA), _dptr(dt))
        d = g.ndim
        return val.value, dA[:d * d].reshape(d, d), dt[:d]

    def affine_register(self, g, fixed, moving, loss, scales, iters, eta, lncc_radius=2):
        """affine_register (affine.hpp:25-30) -> dict(A, t, loss, diverged, iterations)."""
        f, m = as_f64(fixed, g.shape), as_f64(moving, g.shape)
        s = np.ascontiguousarray(scales, dtype=np.float64)
        it = np.ascontiguousarray(iters, dtype=np.int32)
        r = dfm_affine_result()
        self.t.call("affine_register", C.byref(g.c()), _dptr(f), _dptr(m), int(loss), _dptr(s),
                    it.ctypes.data_as(C.POINTER(C.c_int32)), len(s), float(eta),
                    int(lncc_radius), C.byref(r))
        d = g.ndim
        return dict(A=np.array(r.A[:d * d]).reshape(d, d), t=np.array(r.t[:d]), loss=r.loss,
                    diverged=bool(r.diverged), iterations=int(r.iterations))

    def overlap_report(self, g, warped, fixed, gf=None, max_regions=4096):
        """overlap_report (analysis.hpp:67) -> dict(summary..., regions=[dict])."""
        w = np.ascontiguousarray(warped, dtype=np.int32).ravel()
        f = np.ascontiguousarray(fixed, dtype=np.int32).ravel()
        rep = dfm_overlap_summary()
        regs = (dfm_region_overlap * max_regions)()
        self.t.call("overlap_report", C.byref(g.c()), _ipptr(w), C.byref((gf or g).c()),
                    _ipptr(f), C.byref(rep), regs, max_regions)
        out = {k: getattr(rep, k) for k, _ in dfm_overlap_summary._fields_}
        out["regions"] = [{k: getattr(regs[i], k) for k, _ in dfm_region_overlap._fields_}
                          for i in range(min(rep.n_regions, max_regions))]
        return out

    def landmark_error(self, fixed_grid, moving_grid, phi, fixed_mm, moving_mm):
        """landmark_error (analysis.hpp:77-79) -> (distances_mm, mean, max)."""
        phi = as_f64(phi, fixed_grid.field_shape)
        a = np.ascontiguousarray(fixed_mm, dtype=np.float64).reshape(-1, 3)
        b = np.ascontiguousarray(moving_mm, dtype=np.float64).reshape(-1, 3)
        dist = np.zeros(len(a))
        mean, mx = C.c_double(), C.c_double()
        self.t.call("landmark_error", C.byref(fixed_grid.c()), C.byref(moving_grid.c()),
                    C.byref(fixed_grid.c()), _dptr(phi), len(a), _dptr(a), _dptr(b), _dptr(dist),
                    C.byref(mean), C.byref(mx))
        return dist, mean.value, mx.value

    def exp_map(self, g, v, M):
        """exp_map (diffeo.hpp:19-20, diffeo.cpp:66-77): scaling and squaring."""
        v = as_f64(v, g.field_shape)
        out = np.empty(g.field_shape)
        self.t.call("exp_map", C.byref(g.c()), _dptr(v), int(M), _dptr(out))
        return out

    def svf_pullback(self, g, v, grad_phi, M):
        """svf_pullback (diffeo.hpp:22-26, diffeo.cpp:79-167): adjoint of exp_map."""
        v = as_f64(v, g.field_shape)
        gp = as_f64(grad_phi, g.field_shape)
        out = np.empty(g.field_shape)
        self.t.call("svf_pullback", C.byref(g.c()), _dptr(v), _dptr(gp), int(M), _dptr(out))
        return out

    def jacobian_det(self, g, phi):
        phi = as_f64(phi, g.field_shape)
        out = np.empty(g.shape)
        self.t.call("jacobian_det", C.byref(g.c()), _dptr(phi), _dptr(out))
        return out

    def gaussian_smooth(self, g, img, sigma):
        img = as_f64(img, g.shape)
        out = np.empty(g.shape)
        self.t.call("gaussian_smooth", C.byref(g.c()), _dptr(img), _dptr(_sigma3(sigma)),
                    _dptr(out))
        return out

    def gaussian_smooth_field(self, g, f, sigma):
        f = as_f64(f, g.field_shape)
        out = np.empty(g.field_shape)
        self.t.call("gaussian_smooth_field", C.byref(g.c()), _dptr(f), _dptr(_sigma3(sigma)),
                    _dptr(out))
        return out

    def _resample(self, name, g, f, ng):
        f = as_f64(f, g.field_shape)
        out = np.empty(ng.field_shape)
        self.t.call(name, C.byref(g.c()), _dptr(f), C.byref(ng.c()), _dptr(out))
        return out

    def upsample_field(self, g, phi, ng):
        return self._resample("upsample_field", g, phi, ng)

    def resample_field_linear(self, g, f, ng):
        return self._resample("resample_field_linear", g, f, ng)

    def resample_displacement(self, g, phi, ng):
        return self._resample("resample_displacement", g, phi, ng)

    # -- similarity
    def _loss(self, name, fg, fixed, mg, moving, phi, *extra, want_grad=True):
        fixed, moving = as_f64(fixed, fg.shape), as_f64(moving, mg.shape)
        phi = as_f64(phi, fg.field_shape)
        val = C.c_double()
        grad = np.empty(fg.field_shape) if want_grad else None
        self.t.call(name, C.byref(fg.c()), _dptr(fixed), C.byref(mg.c()), _dptr(moving),
                    _dptr(phi), *extra, C.byref(val), _dptr(grad))
        return val.value, grad

    def ssd_eval(self, fg, fixed, phi, moving, mg=None, want_grad=True):
        return self._loss("ssd_eval", fg, fixed, mg or fg, moving, phi, want_grad=want_grad)

    def lncc_eval(self, fg, fixed, phi, moving, radius, mg=None, want_grad=True):
        return self._loss("lncc_eval", fg, fixed, mg or fg, moving, phi, int(radius),
                          want_grad=want_grad)

    def dice_eval(self, fg, fixed, phi, moving, mg=None, want_grad=True):
        return self._loss("dice_eval", fg, fixed, mg or fg, moving, phi, want_grad=want_grad)

    # -- optim
    def adam_step(self, g, m, nu, t, beta1, beta2, eps, v):
        """Returns (dir, m', nu', t') — inputs are not modified."""
        m, nu = as_f64(m, g.field_shape).copy(), as_f64(nu, g.field_shape).copy()
        v = as_f64(v, g.field_shape)
        tt = C.c_int64(int(t))
        out = np.empty(g.field_shape)
        self.t.call("adam_step", C.byref(g.c()), _dptr(m), _dptr(nu), C.byref(tt),
                    float(beta1), float(beta2), float(eps), _dptr(v), _dptr(out))
        return out, m, nu, tt.value

    def upsample_state(self, g, m, nu, ng):
        m, nu = as_f64(m, g.field_shape), as_f64(nu, g.field_shape)
        mo, no = np.empty(ng.field_shape), np.empty(ng.field_shape)
        self.t.call("upsample_state", C.byref(g.c()), _dptr(m), _dptr(nu), C.byref(ng.c()),
                    _dptr(mo), _dptr(no))
        return mo, no

    # -- diffeo
    def eulerian_direction(self, g, grad, phi, use_jac=False):
        grad, phi = as_f64(grad, g.field_shape), as_f64(phi, g.field_shape)
        out = np.empty(g.field_shape)
        self.t.call("eulerian_direction", C.byref(g.c()), _dptr(grad), _dptr(phi),
                    int(bool(use_jac)), _dptr(out))
        return out

    def apply_update(self, g, phi, v, eta, sigma_warp, cap=0.5):
        phi, v = as_f64(phi, g.field_shape), as_f64(v, g.field_shape)
        out = np.empty(g.field_shape)
        self.t.call("apply_update", C.byref(g.c()), _dptr(phi), _dptr(v), float(eta),
                    float(sigma_warp), float(cap), _dptr(out))
        return out

    # -- analysis
    def singularity_fraction(self, g, phi):
        phi = as_f64(phi, g.field_shape)
        v = C.c_double()
        self.t.call("singularity_fraction", C.byref(g.c()), _dptr(phi), C.byref(v))
        return v.value


def make_init(init, ndim: int):
    """RegInit -> dfm_init (keeps referenced arrays alive via the tuple)."""
    ci = dfm_init()
    keep = None
    if init is None:
        ci.kind = INIT_NONE
    elif isinstance(init, AffineTransform):
        ci.kind = INIT_AFFINE
        ci.affine_ndim = init.ndim
        for i, v in enumerate(init.A):
            ci.A[i] = float(v)
        for i, v in enumerate(init.t):
            ci.t[i] = float(v)
    else:
        fg, arr = init
        keep = as_f64(arr, fg.field_shape)
        ci.kind = INIT_FIELD
        ci.field_grid = fg.c()
        ci.field = _dptr(keep)
    return ci, keep


def records_to_log(recs, rl: dfm_runlog) -> RunLog:
    log = RunLog(final_loss=rl.final_loss,
                 final_singularity_fraction=rl.final_singularity_fraction,
                 total_ms=rl.total_ms)
    for i in range(rl.n_records):
        r = recs[i]
        log.iterations.append(IterationRecord(r.scale_index, r.scale, r.iter, r.global_iter,
                                              r.loss, r.max_step, r.wall_ms))
    return log


def schedule_arrays(sched: PyramidSchedule):
    s = np.ascontiguousarray(sched.scales, dtype=np.float64)
    it = np.ascontiguousarray(sched.iterations, dtype=np.int32)
    return s, it
