"""ctypes marshalling for libnseries.so.  Names mirror include/nseries.h one-to-one."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("NSERIES_LIB") or os.path.join(_PKG, "libnseries.so")   # NSERIES_LIB: harness A/B builds

NSERIES_OK = 0
STATUS_NAMES = {
    0: "NSERIES_OK", 1: "NSERIES_ERR_INVALID_ARG", 2: "NSERIES_ERR_UNSUPPORTED_RADIX",
    3: "NSERIES_ERR_PLAN_K_MISMATCH", 4: "NSERIES_ERR_APPROX_TELESCOPE", 5: "NSERIES_ERR_ALIAS",
    6: "NSERIES_ERR_OOM", 7: "NSERIES_ERR_CUDA", 8: "NSERIES_ERR_NO_DEVICE",
    9: "NSERIES_ERR_UNSUPPORTED_SIZE", 10: "NSERIES_ERR_NONFINITE",
}
NSERIES_F64, NSERIES_F32 = 0, 1
NSERIES_PLAN_AUTO, NSERIES_PLAN_BINARY, NSERIES_PLAN_TERNARY, NSERIES_PLAN_RADIX5 = 0, 2, 3, 5
NSERIES_PLAN_RADIX9, NSERIES_PLAN_RADIX15, NSERIES_PLAN_CUSTOM = 9, 15, -1
NSERIES_ELIDE_TRIVIAL = 0x1
NSERIES_ALLOW_APPROX = 0x2
NSERIES_RFORM_TELESCOPE = 0x4
NSERIES_NO_GRAPH = 0x8
NSERIES_SYNC_STATS = 0x10
NSERIES_SYMMETRIC = 0x20
NSERIES_HOST_ASYNC = 0x40
NSERIES_CHECK_FINITE = 0x80
NSERIES_SHARDED_DIRECT = 0x100
NSERIES_MAX_STEPS = 128

# every symbol include/nseries.h declares (tests check the .so exports exactly these)
EXPORTED = [
    "nseries_create", "nseries_destroy", "nseries_status_string", "nseries_version",
    "nseries_plan_build", "nseries_plan_finalize", "nseries_kernel_info", "nseries_eval",
    "nseries_eval_host", "nseries_eval_batched_strided", "nseries_eval_batched",
    "nseries_matmul", "nseries_last_stats", "nseries_solve", "nseries_shard_rows",
    "nseries_comm_unique_id", "nseries_comm_init", "nseries_eval_sharded", "nseries_host_sync",
    "nseries_sharded_arena_bytes", "nseries_peer_export", "nseries_peer_import",
]


class nseries_plan(ctypes.Structure):
    _fields_ = [("n_steps", ctypes.c_int32), ("step", ctypes.c_int32 * NSERIES_MAX_STEPS),
                ("form", ctypes.c_int32 * NSERIES_MAX_STEPS), ("products", ctypes.c_int32),
                ("approx", ctypes.c_int32), ("flags", ctypes.c_uint32), ("k", ctypes.c_int64)]

    @property
    def steps(self):
        return [int(self.step[i]) for i in range(self.n_steps)]

    @property
    def forms(self):
        return [int(self.form[i]) for i in range(self.n_steps)]

    def __repr__(self):
        return f"nseries_plan(k={self.k}, steps={self.steps}, products={self.products}, approx={self.approx})"


class nseries_stats(ctypes.Structure):
    _fields_ = [("products", ctypes.c_int32), ("launches", ctypes.c_int32),
                ("graph_replayed", ctypes.c_int32), ("n_ops", ctypes.c_int32),
                ("ms_total", ctypes.c_float), ("gathers", ctypes.c_int32),
                ("gathers_prefetched", ctypes.c_int32), ("products_paper", ctypes.c_int32),
                ("products_exec", ctypes.c_int32), ("n_steps_timed", ctypes.c_int32),
                ("ms_step", ctypes.c_float * NSERIES_MAX_STEPS), ("nonfinite", ctypes.c_int32)]


class nseries_solve_info(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("products", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("radix", ctypes.c_int32), ("prefix", ctypes.c_int64), ("residual", ctypes.c_double),
                ("history", ctypes.c_double * NSERIES_MAX_STEPS)]


class NSeriesError(RuntimeError):
    def __init__(self, status, where=""):
        self.status = status
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)} ({nseries_status_string(status)})")


_lib = None


def load_library(path=None):
    """Load (never build) libnseries.so; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or _LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"libnseries.so not built at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    plan_p = ctypes.POINTER(nseries_plan)
    sig = {
        "nseries_create": ([ctypes.POINTER(vp), ctypes.c_int], ctypes.c_int),
        "nseries_destroy": ([vp], ctypes.c_int),
        "nseries_status_string": ([ctypes.c_int], ctypes.c_char_p),
        "nseries_version": ([], ctypes.c_char_p),
        "nseries_plan_build": ([i64, ctypes.c_int, ctypes.POINTER(i32), i32, u32, plan_p], ctypes.c_int),
        "nseries_plan_finalize": ([plan_p, i64, u32], ctypes.c_int),
        "nseries_kernel_info": ([i32, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)], ctypes.c_int),
        "nseries_eval": ([vp, vp, i32, i64, plan_p, ctypes.c_int, vp, vp, u32, vp], ctypes.c_int),
        "nseries_eval_host": ([vp, vp, i32, i64, plan_p, ctypes.c_int, vp, vp, u32, vp], ctypes.c_int),
        "nseries_eval_batched_strided": ([vp, vp, i64, i32, i32, i64, plan_p, ctypes.c_int, vp, i64,
                                          u32, vp], ctypes.c_int),
        "nseries_eval_batched": ([vp, vp, i32, i32, i64, plan_p, ctypes.c_int, vp, u32, vp], ctypes.c_int),
        "nseries_matmul": ([vp, ctypes.c_int, vp, vp, vp, i32, vp], ctypes.c_int),
        "nseries_last_stats": ([vp, ctypes.POINTER(nseries_stats)], ctypes.c_int),
        "nseries_solve": ([vp, vp, i32, i32, ctypes.c_double, i32, ctypes.c_int, vp, vp, u32, vp,
                           ctypes.POINTER(nseries_solve_info)], ctypes.c_int),
        "nseries_shard_rows": ([i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)], ctypes.c_int),
        "nseries_comm_unique_id": ([vp], ctypes.c_int),
        "nseries_host_sync": ([vp], ctypes.c_int),
        "nseries_comm_init": ([vp, vp, i32, i32], ctypes.c_int),
        "nseries_eval_sharded": ([vp, ctypes.POINTER(vp), i32, i32, i32, i32, i64, plan_p, ctypes.c_int,
                                  ctypes.POINTER(vp), ctypes.POINTER(vp), u32, vp], ctypes.c_int),
        "nseries_sharded_arena_bytes": ([i32, i32, i32, i64, plan_p, u32, i32, ctypes.POINTER(ctypes.c_uint64)],
                                        ctypes.c_int),
        "nseries_peer_export": ([vp, ctypes.c_uint64, vp], ctypes.c_int),
        "nseries_peer_import": ([vp, vp, i32], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(st, where):
    if st != NSERIES_OK:
        raise NSeriesError(st, where)


def _ptr(x):
    """Device/host pointer of a torch tensor, numpy array or raw int (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dtype_of(t):
    name = str(getattr(t, "dtype", ""))
    if name.endswith("float64"):
        return NSERIES_F64
    if name.endswith("float32"):
        return NSERIES_F32
    raise TypeError(f"unsupported dtype {name}")


# ---------------------------------------------------------------- 1:1 wrappers

def nseries_status_string(status):
    return load_library().nseries_status_string(int(status)).decode()


def nseries_version():
    return load_library().nseries_version().decode()


def nseries_create(device=0):
    h = ctypes.c_void_p()
    _check(load_library().nseries_create(ctypes.byref(h), int(device)), "nseries_create")
    return h


def nseries_destroy(h):
    _check(load_library().nseries_destroy(h), "nseries_destroy")


def nseries_plan_build(k, kind=NSERIES_PLAN_AUTO, radices=None, flags=0):
    p = nseries_plan()
    arr, n = None, 0
    if radices:
        n = len(radices)
        arr = (ctypes.c_int32 * n)(*radices)
    _check(load_library().nseries_plan_build(int(k), int(kind), arr, n, int(flags), ctypes.byref(p)),
           "nseries_plan_build")
    return p


def nseries_plan_finalize(steps, k, flags=0):
    p = nseries_plan()
    p.n_steps = len(steps)
    for i, s in enumerate(steps):
        p.step[i] = int(s)
    _check(load_library().nseries_plan_finalize(ctypes.byref(p), int(k), int(flags)), "nseries_plan_finalize")
    return p


def nseries_kernel_info(m):
    mu, ex, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(0)
    L = load_library()
    _check(L.nseries_kernel_info(int(m), ctypes.byref(mu), ctypes.byref(ex), None, ctypes.byref(n)),
           "nseries_kernel_info")
    buf = (ctypes.c_double * n.value)()
    _check(L.nseries_kernel_info(int(m), ctypes.byref(mu), ctypes.byref(ex), buf, ctypes.byref(n)),
           "nseries_kernel_info")
    return {"mu": mu.value, "exact": bool(ex.value), "coeffs": list(buf)}


def nseries_eval(h, A, d, k, plan=None, dtype=None, S=None, R_out=None, flags=0, stream=None):
    dt = _dtype_of(A) if dtype is None else dtype
    st = load_library().nseries_eval(h, _ptr(A), int(d), int(k), ctypes.byref(plan) if plan is not None else None,
                                     dt, _ptr(S), _ptr(R_out), int(flags), _stream(stream))
    _check(st, "nseries_eval")


def nseries_eval_host(h, A, d, k, plan=None, dtype=None, S=None, R_out=None, flags=0, stream=None):
    dt = _dtype_of(A) if dtype is None else dtype
    st = load_library().nseries_eval_host(h, _ptr(A), int(d), int(k),
                                          ctypes.byref(plan) if plan is not None else None,
                                          dt, _ptr(S), _ptr(R_out), int(flags), _stream(stream))
    _check(st, "nseries_eval_host")


def nseries_host_sync(h):
    """Wait for every NSERIES_HOST_ASYNC nseries_eval_host call on this handle."""
    _check(load_library().nseries_host_sync(h), "nseries_host_sync")


def nseries_eval_batched_strided(h, A, strideA, batch, d, k, plan=None, dtype=None, S=None,
                                 strideS=None, flags=0, stream=None):
    dt = _dtype_of(A) if dtype is None else dtype
    strideS = strideA if strideS is None else strideS
    st = load_library().nseries_eval_batched_strided(
        h, _ptr(A), int(strideA), int(batch), int(d), int(k),
        ctypes.byref(plan) if plan is not None else None, dt, _ptr(S), int(strideS), int(flags),
        _stream(stream))
    _check(st, "nseries_eval_batched_strided")


def nseries_eval_batched(h, A_ptrs, batch, d, k, plan=None, dtype=NSERIES_F32, S_ptrs=None, flags=0,
                         stream=None):
    st = load_library().nseries_eval_batched(h, _ptr(A_ptrs), int(batch), int(d), int(k),
                                             ctypes.byref(plan) if plan is not None else None,
                                             int(dtype), _ptr(S_ptrs), int(flags), _stream(stream))
    _check(st, "nseries_eval_batched")


def nseries_matmul(h, X, Y, C, d, dtype=None, stream=None):
    dt = _dtype_of(X) if dtype is None else dtype
    _check(load_library().nseries_matmul(h, dt, _ptr(X), _ptr(Y), _ptr(C), int(d), _stream(stream)),
           "nseries_matmul")


def nseries_solve(h, A, d, m, tol, max_steps=NSERIES_MAX_STEPS, Y=None, R_out=None, flags=0, stream=None,
                  dtype=None):
    dt = _dtype_of(A) if dtype is None else dtype
    info = nseries_solve_info()
    _check(load_library().nseries_solve(h, _ptr(A), int(d), int(m), float(tol), int(max_steps), dt, _ptr(Y),
                                        _ptr(R_out), int(flags), _stream(stream), ctypes.byref(info)),
           "nseries_solve")
    return {"steps": info.steps, "products": info.products, "converged": bool(info.converged),
            "radix": info.radix, "prefix": info.prefix, "residual": info.residual,
            "history": [info.history[i] for i in range(info.steps)]}


def nseries_shard_rows(d, nshards, shard):
    """(row0, rows) of row block `shard` of `nshards` over d rows (host-only)."""
    r0, n = ctypes.c_int32(), ctypes.c_int32()
    _check(load_library().nseries_shard_rows(int(d), int(nshards), int(shard), ctypes.byref(r0), ctypes.byref(n)),
           "nseries_shard_rows")
    return r0.value, n.value


def nseries_comm_unique_id():
    """128-byte NCCL unique id (rank 0 creates it, the caller ships it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().nseries_comm_unique_id(buf), "nseries_comm_unique_id")
    return buf.raw


def nseries_comm_init(h, uid, nranks, rank):
    if len(uid) != 128:
        raise ValueError("NCCL unique id must be 128 bytes")
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(load_library().nseries_comm_init(h, buf, int(nranks), int(rank)), "nseries_comm_init")


def nseries_sharded_arena_bytes(d, nshards, n_local, k, plan=None, flags=0, want_R=False):
    """Arena bytes one rank needs for NSERIES_SHARDED_DIRECT across processes (host-only)."""
    b = ctypes.c_uint64()
    _check(load_library().nseries_sharded_arena_bytes(int(d), int(nshards), int(n_local), int(k),
                                                      ctypes.byref(plan) if plan is not None else None,
                                                      int(flags), int(bool(want_R)), ctypes.byref(b)),
           "nseries_sharded_arena_bytes")
    return b.value


def nseries_peer_export(h, nbytes):
    """Allocate / grow the handle's arena to nbytes; returns its 64-byte CUDA IPC handle."""
    buf = ctypes.create_string_buffer(64)
    _check(load_library().nseries_peer_export(h, ctypes.c_uint64(int(nbytes)), buf), "nseries_peer_export")
    return buf.raw


def nseries_peer_import(h, handles):
    """Map the peers' arenas: `handles` = list of 64-byte IPC handles indexed by rank."""
    blob = b"".join(bytes(x) for x in handles)
    if any(len(x) != 64 for x in handles):
        raise ValueError("IPC handles are 64 bytes")
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(load_library().nseries_peer_import(h, buf, len(handles)), "nseries_peer_import")


def nseries_eval_sharded(h, A_shards, first_shard, nshards, d, k, plan=None, S_shards=None, R_shards=None,
                         flags=0, stream=None, dtype=NSERIES_F64):
    """Row-sharded evaluation: A_shards / S_shards (/ R_shards) are lists of this process's row
    blocks (device tensors), shards first_shard .. first_shard + len - 1 of nshards."""
    n = len(A_shards)
    arr = ctypes.c_void_p * n
    a = arr(*[_ptr(x) for x in A_shards])
    s_ = arr(*[_ptr(x) for x in S_shards])
    r = arr(*[_ptr(x) for x in R_shards]) if R_shards is not None else None
    st = load_library().nseries_eval_sharded(h, a, n, int(first_shard), int(nshards), int(d), int(k),
                                             ctypes.byref(plan) if plan is not None else None, int(dtype), s_, r,
                                             int(flags), _stream(stream))
    _check(st, "nseries_eval_sharded")


def nseries_last_stats(h):
    s = nseries_stats()
    _check(load_library().nseries_last_stats(h, ctypes.byref(s)), "nseries_last_stats")
    return {"products": s.products, "launches": s.launches, "graph_replayed": s.graph_replayed,
            "n_ops": s.n_ops, "ms_total": s.ms_total, "gathers": s.gathers,
            "gathers_prefetched": s.gathers_prefetched, "products_paper": s.products_paper,
            "products_exec": s.products_exec, "ms_step": [s.ms_step[i] for i in range(s.n_steps_timed)],
            "nonfinite": s.nonfinite}


__all__ = [n for n in dir() if n.startswith(("nseries_", "NSERIES_"))] + [
    "NSeriesError", "load_library", "EXPORTED", "STATUS_NAMES"]
