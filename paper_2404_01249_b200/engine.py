"""Python host-side mirror of the difform:: API over the CUDA C-ABI.

This is the thin Python face of libdifform_cuda.so (the product is the .so and
its C-ABI, include/difform_gpu.h); tests and bench.py call through it.  There
is NO CPU fallback: constructing a Context without the built library or without
a CUDA device raises.

    ctx = Context(device=0, precision="f32")
    phi, log = ctx.register_images(grid, fixed, moving, cfg, schedule)
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _abi as A

LIB_PATH = os.environ.get(  # DFM_LIB: an alternative build (tuning A/B only)
    "DFM_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdifform_cuda.so"))

# every entry point include/difform_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "dfm_abi_version", "dfm_config_defaults", "dfm_ctx_create", "dfm_ctx_destroy",
    "dfm_ctx_precision", "dfm_ctx_stream", "dfm_last_error", "dfm_ctx_launch_count",
    "dfm_validate_grid", "dfm_downsample_grid", "dfm_downsample_image",
    "dfm_sample_linear_points", "dfm_warp_image", "dfm_warp_labels", "dfm_compose",
    "dfm_jacobian_det", "dfm_gaussian_smooth", "dfm_gaussian_smooth_field",
    "dfm_upsample_field", "dfm_resample_field_linear", "dfm_resample_displacement",
    "dfm_ssd_eval", "dfm_lncc_eval", "dfm_dice_eval", "dfm_adam_step", "dfm_upsample_state",
    "dfm_eulerian_direction", "dfm_apply_update", "dfm_singularity_fraction", "dfm_register",
    "dfm_dev_register", "dfm_ctx_set_profiling", "dfm_ctx_kernel_times",
    "dfm_slab_bounds", "dfm_slab_halo", "dfm_slab_unique_id", "dfm_dev_register_slab",
    "dfm_ctx_set_option", "dfm_exp_map", "dfm_svf_pullback", "dfm_affine_to_field",
    "dfm_affine_param_gradient", "dfm_affine_register", "dfm_overlap_report",
    "dfm_dev_overlap_report", "dfm_dev_warp_labels", "dfm_landmark_error", "dfm_sweep",
    "dfm_mhd_read_header", "dfm_mhd_write_image", "dfm_mhd_read_image", "dfm_mhd_write_labels",
    "dfm_mhd_read_labels", "dfm_mhd_write_field", "dfm_mhd_read_field", "dfm_dev_load_image_mhd",
    "dfm_dev_save_field_mhd", "dfm_ctx_debug_read", "dfm_sample_field_points", "dfm_jacobian",
    "dfm_upsample_field_cubic", "dfm_sgd_step", "dfm_validate_config", "dfm_validate_schedule",
    "dfm_dev_register_slab_tp",
]

OPT_BRICK_MAX = 1
OPT_FORCE_LEGACY = 2
OPT_PERSIST = 3
OPT_PDL = 4
OPT_SPLIT = 5
OPT_SPLIT_FOLD_MAX = 6
OPT_LARGE_MIN = 7
OPT_SLAB_REPL_MAX = 9
OPT_SLAB_OVERLAP = 10
OPT_EXACT = 11
OPT_NARROW = 12

_lib: Optional[C.CDLL] = None

# dfm_slab_transport (difform_gpu.h): host callbacks of a caller transport
_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                        C.c_int64)
_SUM_F64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
_MAX_U64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int64)
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                         C.POINTER(C.c_int64))


class SlabTransportC(C.Structure):
    _fields_ = [("user", C.c_void_p), ("sendrecv", _SENDRECV), ("allreduce_sum_f64", _SUM_F64),
                ("allreduce_max_u64", _MAX_U64), ("allgather", _ALLGATHER)]


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads (once) the in-tree CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: build it with `python -m paper_2404_01249_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(path)
        lib.dfm_ctx_create.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        lib.dfm_ctx_create.restype = C.c_int
        lib.dfm_ctx_destroy.argtypes = [C.c_void_p]
        lib.dfm_ctx_destroy.restype = None
        lib.dfm_ctx_stream.argtypes = [C.c_void_p]
        lib.dfm_ctx_stream.restype = C.c_void_p
        lib.dfm_ctx_launch_count.argtypes = [C.c_void_p]
        lib.dfm_ctx_launch_count.restype = C.c_int64
        lib.dfm_ctx_precision.argtypes = [C.c_void_p]
        lib.dfm_ctx_precision.restype = C.c_int
        lib.dfm_abi_version.restype = C.c_int
        lib.dfm_config_defaults.argtypes = [C.POINTER(A.dfm_config)]
        lib.dfm_config_defaults.restype = None
        lib.dfm_validate_grid.argtypes = [C.POINTER(A.dfm_grid)]
        lib.dfm_validate_grid.restype = C.c_int
        lib.dfm_downsample_grid.argtypes = [C.POINTER(A.dfm_grid), C.POINTER(C.c_double),
                                            C.POINTER(A.dfm_grid)]
        lib.dfm_downsample_grid.restype = C.c_int
        lib.dfm_ctx_set_profiling.argtypes = [C.c_void_p, C.c_int]
        lib.dfm_ctx_set_profiling.restype = C.c_int
        lib.dfm_dev_warp_labels.argtypes = [C.c_void_p, C.POINTER(A.dfm_grid), C.c_void_p,
                                            C.c_void_p, C.c_void_p]
        lib.dfm_dev_warp_labels.restype = C.c_int
        lib.dfm_dev_overlap_report.argtypes = [
            C.c_void_p, C.POINTER(A.dfm_grid), C.c_void_p, C.c_void_p,
            C.POINTER(A.dfm_overlap_summary), C.POINTER(A.dfm_region_overlap), C.c_int64]
        lib.dfm_dev_overlap_report.restype = C.c_int
        lib.dfm_dev_load_image_mhd.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(A.dfm_grid),
                                               C.c_void_p]
        lib.dfm_dev_save_field_mhd.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(A.dfm_grid),
                                               C.c_void_p]
        lib.dfm_ctx_set_option.argtypes = [C.c_void_p, C.c_int, C.c_int64]
        lib.dfm_ctx_set_option.restype = C.c_int
        lib.dfm_ctx_kernel_times.argtypes = [C.c_void_p, C.POINTER(C.c_double),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.dfm_ctx_kernel_times.restype = C.c_int
        lib.dfm_ctx_debug_read.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.c_size_t,
                                           C.c_void_p]
        lib.dfm_ctx_debug_read.restype = C.c_int
        reg = [C.c_void_p, C.POINTER(A.dfm_grid), C.c_void_p, C.c_void_p]
        lib.dfm_register.argtypes = reg + [C.c_int, C.POINTER(A.dfm_config),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                           C.c_int32, C.POINTER(A.dfm_init), C.c_void_p, C.c_int,
                                           C.POINTER(A.dfm_iter_record), C.c_int64,
                                           C.POINTER(A.dfm_runlog)]
        lib.dfm_register.restype = C.c_int
        lib.dfm_dev_register.argtypes = reg + [C.POINTER(A.dfm_config), C.POINTER(C.c_double),
                                               C.POINTER(C.c_int32), C.c_int32, C.c_void_p,
                                               C.POINTER(A.dfm_iter_record), C.c_int64,
                                               C.POINTER(A.dfm_runlog)]
        lib.dfm_dev_register.restype = C.c_int
        lib.dfm_slab_bounds.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_int64)]
        lib.dfm_slab_bounds.restype = C.c_int
        lib.dfm_slab_halo.argtypes = [C.POINTER(A.dfm_config), C.POINTER(A.dfm_grid)]
        lib.dfm_slab_halo.restype = C.c_int
        lib.dfm_slab_unique_id.argtypes = [C.c_char_p]
        lib.dfm_slab_unique_id.restype = C.c_int
        lib.dfm_dev_register_slab.argtypes = reg + [
            C.POINTER(A.dfm_config), C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int32,
            C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_void_p, C.POINTER(C.c_int64),
            C.POINTER(C.c_int64), C.POINTER(A.dfm_iter_record), C.c_int64,
            C.POINTER(A.dfm_runlog)]
        lib.dfm_dev_register_slab.restype = C.c_int
        lib.dfm_dev_register_slab_tp.argtypes = reg + [
            C.POINTER(A.dfm_config), C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int32,
            C.c_int, C.c_int, C.POINTER(SlabTransportC), C.c_void_p, C.POINTER(C.c_int64),
            C.POINTER(C.c_int64), C.POINTER(A.dfm_iter_record), C.c_int64,
            C.POINTER(A.dfm_runlog)]
        lib.dfm_dev_register_slab_tp.restype = C.c_int
        _lib = lib
    return _lib


KCLASS_NAMES = ["loss_fwd", "lncc_bwd", "smooth_adam", "compose_smooth", "monitor", "pyramid",
                "epilogue"]


class Context(A.HostAPI):
    """A dfm_ctx: one CUDA stream + workspace on `device`, fp32 or fp64."""

    def __init__(self, device: int = 0, precision: str = "f32"):
        lib = load_library()
        prec = {"f32": A.PREC_F32, "f64": A.PREC_F64}[precision]
        h = C.c_void_p()
        tbl = A.CallTable(lib, "dfm_", ctx=None)
        tbl.check(lib.dfm_ctx_create(device, prec, C.byref(h)), "dfm_ctx_create")
        super().__init__(A.CallTable(lib, "dfm_", ctx=h))
        self.lib = lib
        self.handle = h
        self.precision = precision
        self.device = device

    def close(self):
        if self.handle:
            self.lib.dfm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        return int(self.lib.dfm_ctx_stream(self.handle) or 0)

    @property
    def launch_count(self) -> int:
        return int(self.lib.dfm_ctx_launch_count(self.handle))

    def set_profiling(self, on: bool):
        self.t.check(self.lib.dfm_ctx_set_profiling(self.handle, int(on)), "set_profiling")

    def set_option(self, key: int, value: int):
        """dfm_ctx_set_option: OPT_BRICK_MAX (voxels) / OPT_FORCE_LEGACY (0|1)."""
        self.t.check(self.lib.dfm_ctx_set_option(self.handle, int(key), int(value)),
                     "set_option")

    def debug_read(self, name: str, count: int, offset: int = 0) -> np.ndarray:
        """dfm_ctx_debug_read: `count` elements (context precision) of the named
        workspace buffer from element `offset` (white-box parity tests)."""
        dt = np.float64 if self.precision == "f64" else np.float32
        out = np.empty(int(count), dtype=dt)
        it = out.itemsize
        self.t.check(self.lib.dfm_ctx_debug_read(self.handle, name.encode(), int(offset) * it,
                                                 out.nbytes, out.ctypes.data), "debug_read")
        return out

    def debug_field(self, name: str, g: A.GridMeta) -> np.ndarray:
        """A 3-plane SoA workspace field packed at g's voxel count -> AoS
        (z, y, x, 3) float64, the host layout of the reference."""
        n = g.voxel_count
        soa = self.debug_read(name, 3 * n).astype(np.float64).reshape(3, n)
        return np.ascontiguousarray(soa.T).reshape(g.field_shape)

    def kernel_times(self) -> dict:
        ms = (C.c_double * A.NUM_KCLASS)()
        n = (C.c_int64 * A.NUM_KCLASS)()
        v = (C.c_int64 * A.NUM_KCLASS)()
        self.t.check(self.lib.dfm_ctx_kernel_times(self.handle, ms, n, v), "kernel_times")
        return {KCLASS_NAMES[k]: {"ms": ms[k], "launches": n[k], "voxels": v[k]}
                for k in range(A.NUM_KCLASS)}

    # -- pipeline
    def register_images(self, g: A.GridMeta, fixed, moving, cfg: A.RegistrationConfig,
                        sched: A.PyramidSchedule, init=None, field_dtype=np.float64):
        """register_images (pipeline.hpp:70-73) with HOST arrays -> (field, RunLog).

        fixed/moving may be float32 or float64 numpy arrays (float32 halves the
        host->device bytes); the field comes back as AoS ``field_dtype``.
        """
        img_dt = np.float32 if np.asarray(fixed).dtype == np.float32 else np.float64
        f = np.ascontiguousarray(fixed, dtype=img_dt).reshape(g.shape)
        m = np.ascontiguousarray(moving, dtype=img_dt).reshape(g.shape)
        s, it = A.schedule_arrays(sched)
        cap = int(it.sum()) + 1
        recs = (A.dfm_iter_record * cap)()
        rl = A.dfm_runlog()
        out = np.empty(g.field_shape, dtype=field_dtype)
        ci, keep = A.make_init(init, g.ndim)
        cc = cfg.c()
        rc = self.lib.dfm_register(
            self.handle, C.byref(g.c()), f.ctypes.data, m.ctypes.data,
            A.HOST_F32 if img_dt == np.float32 else A.HOST_F64, C.byref(cc), A._dptr(s),
            it.ctypes.data_as(C.POINTER(C.c_int32)), len(s), C.byref(ci), out.ctypes.data,
            A.HOST_F32 if field_dtype == np.float32 else A.HOST_F64, recs, cap, C.byref(rl))
        self.t.check(rc, "register")
        del keep
        return out, A.records_to_log(recs, rl)

    def register_device(self, g: A.GridMeta, d_fixed: int, d_moving: int,
                        cfg: A.RegistrationConfig, sched: A.PyramidSchedule,
                        d_out: int = 0):
        """dfm_dev_register: device pointers (context precision), SoA result."""
        s, it = A.schedule_arrays(sched)
        cap = int(it.sum()) + 1
        recs = (A.dfm_iter_record * cap)()
        rl = A.dfm_runlog()
        cc = cfg.c()
        rc = self.lib.dfm_dev_register(self.handle, C.byref(g.c()), C.c_void_p(d_fixed),
                                       C.c_void_p(d_moving), C.byref(cc), A._dptr(s),
                                       it.ctypes.data_as(C.POINTER(C.c_int32)), len(s),
                                       C.c_void_p(d_out) if d_out else None, recs, cap,
                                       C.byref(rl))
        self.t.check(rc, "dev_register")
        return A.records_to_log(recs, rl)


def slab_bounds(nz: int, part: int, nparts: int, halo: int):
    """(zlo, zhi, hlo, hhi) of slab `part` — the plan every rank computes."""
    lib = load_library()
    out = (C.c_int64 * 4)()
    rc = lib.dfm_slab_bounds(int(nz), int(part), int(nparts), int(halo), out)
    if rc != A.DFM_OK:
        raise A.InvalidArgument("slab_bounds: bad arguments")
    return tuple(int(v) for v in out)


def slab_halo(cfg: A.RegistrationConfig) -> int:
    lib = load_library()
    cc = cfg.c()
    return int(lib.dfm_slab_halo(C.byref(cc), None))


def slab_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    rc = lib.dfm_slab_unique_id(buf)
    if rc != A.DFM_OK:
        raise A.DeviceError("dfm_slab_unique_id failed")
    return buf.raw


def register_slab(ctx: "Context", g: A.GridMeta, d_fixed: int, d_moving: int,
                  cfg: A.RegistrationConfig, sched: A.PyramidSchedule, rank: int = 0,
                  world: int = 1, nccl_id: bytes = None, emulate: int = 1, d_out: int = 0):
    """dfm_dev_register_slab: z-slab decomposed registration -> (zlo, zhi, RunLog)."""
    s, it = A.schedule_arrays(sched)
    cap = int(it.sum()) + 1
    recs = (A.dfm_iter_record * cap)()
    rl = A.dfm_runlog()
    cc = cfg.c()
    zlo, zhi = C.c_int64(), C.c_int64()
    rc = ctx.lib.dfm_dev_register_slab(
        ctx.handle, C.byref(g.c()), C.c_void_p(d_fixed), C.c_void_p(d_moving), C.byref(cc),
        A._dptr(s), it.ctypes.data_as(C.POINTER(C.c_int32)), len(s), rank, world, nccl_id,
        emulate, C.c_void_p(d_out) if d_out else None, C.byref(zlo), C.byref(zhi), recs, cap,
        C.byref(rl))
    ctx.t.check(rc, "register_slab")
    return zlo.value, zhi.value, A.records_to_log(recs, rl)


class TorchDistTransport:
    """dfm_slab_transport over torch.distributed (any backend with CPU tensors,
    e.g. gloo): the host-staged collectives of a slab decomposition between
    processes — no NCCL needed, so two ranks may share one GPU."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

        def _bytes(ptr, n):
            import torch
            a = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(int(n),))
            return torch.from_numpy(a)

        def sendrecv(_, peer, sbuf, sbytes, rbuf, rbytes):
            try:
                s = _bytes(sbuf, sbytes)
                r = _bytes(rbuf, rbytes)
                reqs = [dist.isend(s, peer, group=group), dist.irecv(r, peer, group=group)]
                for q in reqs:
                    q.wait()
                return 0
            except Exception:  # noqa: BLE001 - reported as a status code
                return 1

        def sum_f64(_, buf, n):
            try:
                import torch
                t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(int(n),)))
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def max_u64(_, buf, n):
            try:
                import torch
                a = np.ctypeslib.as_array(buf, shape=(int(n),))
                t = torch.from_numpy(a.view(np.int64))  # < 2^63 here: same order
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def allgather(_, sbuf, sbytes, rbuf, counts):
            try:
                import torch
                world = dist.get_world_size(group)
                cnt = [int(counts[r]) for r in range(world)]
                mx = max(cnt)
                s = torch.zeros(mx, dtype=torch.uint8)
                s[:int(sbytes)] = _bytes(sbuf, sbytes)
                outs = [torch.empty(mx, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, s, group=group)
                r = _bytes(rbuf, sum(cnt))
                off = 0
                for k in range(world):
                    r[off:off + cnt[k]] = outs[k][:cnt[k]]
                    off += cnt[k]
                return 0
            except Exception:  # noqa: BLE001
                return 1

        # keep the ctypes callbacks alive as long as the transport
        self._cb = (_SENDRECV(sendrecv), _SUM_F64(sum_f64), _MAX_U64(max_u64),
                    _ALLGATHER(allgather))
        self.c = SlabTransportC(None, *self._cb)


def register_slab_tp(ctx: "Context", g: A.GridMeta, d_fixed: int, d_moving: int,
                     cfg: A.RegistrationConfig, sched: A.PyramidSchedule, rank: int, world: int,
                     transport: TorchDistTransport, d_out: int = 0):
    """dfm_dev_register_slab_tp: this process = slab `rank` of `world`, every
    collective through `transport` -> (zlo, zhi, RunLog)."""
    s, it = A.schedule_arrays(sched)
    cap = int(it.sum()) + 1
    recs = (A.dfm_iter_record * cap)()
    rl = A.dfm_runlog()
    cc = cfg.c()
    zlo, zhi = C.c_int64(), C.c_int64()
    rc = ctx.lib.dfm_dev_register_slab_tp(
        ctx.handle, C.byref(g.c()), C.c_void_p(d_fixed), C.c_void_p(d_moving), C.byref(cc),
        A._dptr(s), it.ctypes.data_as(C.POINTER(C.c_int32)), len(s), rank, world,
        C.byref(transport.c), C.c_void_p(d_out) if d_out else None, C.byref(zlo), C.byref(zhi),
        recs, cap, C.byref(rl))
    ctx.t.check(rc, "register_slab_tp")
    return zlo.value, zhi.value, A.records_to_log(recs, rl)


def cuda_available() -> bool:
    """True when a CUDA device is visible (checked without torch)."""
    try:
        rt = C.CDLL("libcuda.so.1")
    except OSError:
        return False
    n = C.c_int(0)
    if rt.cuInit(0) != 0:
        return False
    return rt.cuDeviceGetCount(C.byref(n)) == 0 and n.value > 0
