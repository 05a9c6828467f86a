"""Thin ctypes binding of libbdeg.so (include/bdeg.h) — argument marshalling
only.  Every step of the degree computation runs in the library: the C++
front end (Smith form, P_0, point configuration, planner) and the sm_100a
kernels.  There is no Python or CPU fallback: if libbdeg.so is missing the
import fails, and device entry points raise BdegError(BDEG_E_CUDA) without
a B200.

PyTorch is used only as plumbing: device workspace (a torch.uint8 CUDA
tensor), the current CUDA stream, and torch.distributed for the multi-GPU
all-reduce (see bench.py / multi.py).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BDEG_LIB") or os.path.join(_HERE, "libbdeg.so")  # BDEG_LIB: tuning builds

BDEG_OK = 0
BDEG_E_INVALID = 1
BDEG_E_INCONSISTENT = 2
BDEG_E_DEGENERATE = 3
BDEG_E_IO = 4
BDEG_E_TOO_LARGE = 5
BDEG_E_CUDA = 6
BDEG_E_COMM = 7

FLAG_NO_LLL = 0x1
FLAG_NO_HOMOG_SHORTCUT = 0x2
FLAG_FORCE_TIER0 = 0x4
FLAG_FORCE_TIER1 = 0x8
FLAG_NO_RELIFT = 0x10
FLAG_FORCE_TIER2 = 0x20
FLAG_DEGREE_ONLY = 0x40
FLAG_NATURAL_ORDER = 0x80      # system plans: first-occurrence point order (default: sorted by lifting residual)
TIER_DTYPE = {0: "int32", 1: "int32/int64", 2: "int64/int128", 4: "int128/int256"}

NSLOTS = 16


class BdegError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"bdeg error {status}: {msg}")
        self.status = status


class _Problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32),
                ("A", ctypes.POINTER(ctypes.c_int64)),
                ("b_re", ctypes.POINTER(ctypes.c_double)),
                ("b_im", ctypes.POINTER(ctypes.c_double)),
                ("lifting", ctypes.POINTER(ctypes.c_int64))]


class _Options(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("lift_bits", ctypes.c_int32),
                ("max_relift", ctypes.c_int32), ("device", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("flags", ctypes.c_uint32),
                ("inner_levels", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32)]


class _Result(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("rank", ctypes.c_int32), ("dim", ctypes.c_int32),
                ("K", ctypes.c_int32), ("N", ctypes.c_int32), ("tier", ctypes.c_int32),
                ("homogeneous", ctypes.c_int32), ("inner_levels", ctypes.c_int32),
                ("comp_lo", ctypes.c_uint64), ("comp_hi", ctypes.c_uint64),
                ("deg_lo", ctypes.c_uint64), ("deg_hi", ctypes.c_int64),
                ("candidates", ctypes.c_uint64), ("cells", ctypes.c_uint64),
                ("singular", ctypes.c_uint64), ("ties", ctypes.c_uint64),
                ("overflow_reruns", ctypes.c_uint64), ("updates", ctypes.c_uint64),
                ("leaves", ctypes.c_uint64), ("dead_leaves", ctypes.c_uint64),
                ("relifts", ctypes.c_int32),
                ("consistent", ctypes.c_int32), ("singular_complete", ctypes.c_int32),
                ("seed_used", ctypes.c_uint64),
                ("total_candidates", ctypes.c_uint64),
                ("plan_ms", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("wide_reruns", ctypes.c_uint64),
                ("dead_full", ctypes.c_int32)]


_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32)
_A2A_COUNTS = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                               ctypes.POINTER(ctypes.c_uint64))
_A2A_CELLS = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                              ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64))


class _Comm(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allreduce_sum", _ALLREDUCE),
                ("alltoall_counts", _A2A_COUNTS), ("alltoall_cells", _A2A_CELLS)]


EXPORTS = ["bdeg_default_options", "bdeg_plan", "bdeg_plan_points", "bdeg_plan_info",
           "bdeg_workspace_bytes", "bdeg_set_workspace", "bdeg_degree", "bdeg_degree_range",
           "bdeg_degree_partial", "bdeg_finalize", "bdeg_relift", "bdeg_last_error",
           "bdeg_status_str", "bdeg_destroy", "bdeg_launch_count", "bdeg_num_items",
           "bdeg_item_range", "bdeg_cells", "bdeg_degree_walk", "bdeg_cell_normal",
           "bdeg_steal_create", "bdeg_steal_attach", "bdeg_rank_modp", "bdeg_dimension_modp",
           "bdeg_plan_points_get", "bdeg_queue_info", "bdeg_smith_gpu", "bdeg_degree_walk_sharded"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(libbdeg has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    if os.environ.get("BDEG_LIB"):
        # A/B tuning builds of older revisions may lack the newest entry points
        class _Tolerant:
            def __init__(self, l):
                object.__setattr__(self, "_l", l)

            def __getattr__(self, name):
                try:
                    return getattr(self._l, name)
                except AttributeError:
                    return type("_Missing", (), {})()

        lib = _Tolerant(lib)
    P = ctypes.POINTER
    plan_t = ctypes.c_void_p
    lib.bdeg_default_options.argtypes = [P(_Options)]
    lib.bdeg_default_options.restype = None
    lib.bdeg_plan.argtypes = [P(_Problem), P(_Options), P(plan_t)]
    lib.bdeg_plan_points.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int64),
                                     P(ctypes.c_int64), P(_Options), P(plan_t)]
    lib.bdeg_plan_info.argtypes = [plan_t, P(_Result)]
    lib.bdeg_plan_points_get.argtypes = [plan_t, P(ctypes.c_int64), P(ctypes.c_int64)]
    lib.bdeg_workspace_bytes.argtypes = [plan_t]
    lib.bdeg_workspace_bytes.restype = ctypes.c_size_t
    lib.bdeg_set_workspace.argtypes = [plan_t, ctypes.c_void_p, ctypes.c_size_t]
    lib.bdeg_degree.argtypes = [plan_t, P(_Result)]
    lib.bdeg_degree_range.argtypes = [plan_t, ctypes.c_uint64, ctypes.c_uint64, P(_Result)]
    lib.bdeg_degree_partial.argtypes = [plan_t, ctypes.c_void_p]
    lib.bdeg_finalize.argtypes = [plan_t, P(ctypes.c_int64), P(_Result)]
    lib.bdeg_relift.argtypes = [plan_t, ctypes.c_int32]
    lib.bdeg_last_error.argtypes = [plan_t]
    lib.bdeg_last_error.restype = ctypes.c_char_p
    lib.bdeg_status_str.argtypes = [ctypes.c_int]
    lib.bdeg_status_str.restype = ctypes.c_char_p
    lib.bdeg_destroy.argtypes = [plan_t]
    lib.bdeg_destroy.restype = None
    lib.bdeg_num_items.argtypes = [plan_t]
    lib.bdeg_num_items.restype = ctypes.c_uint64
    lib.bdeg_item_range.argtypes = [plan_t, ctypes.c_uint64, P(ctypes.c_uint64), P(ctypes.c_uint64)]
    lib.bdeg_item_range.restype = ctypes.c_int
    lib.bdeg_queue_info.argtypes = [plan_t, P(ctypes.c_uint64), P(ctypes.c_uint64), P(ctypes.c_uint64),
                                    P(ctypes.c_uint64)]
    lib.bdeg_queue_info.restype = ctypes.c_int
    lib.bdeg_cells.argtypes = [plan_t, ctypes.c_uint64, ctypes.c_uint64, P(ctypes.c_uint64),
                               ctypes.c_uint64, P(ctypes.c_uint64)]
    lib.bdeg_cells.restype = ctypes.c_int
    lib.bdeg_degree_walk.argtypes = [plan_t, P(_Result)]
    lib.bdeg_cell_normal.argtypes = [plan_t, ctypes.c_uint64, ctypes.c_uint64, P(ctypes.c_int64),
                                     P(ctypes.c_int64)]
    lib.bdeg_cell_normal.restype = ctypes.c_int
    lib.bdeg_degree_walk.restype = ctypes.c_int
    lib.bdeg_degree_walk_sharded.argtypes = [plan_t, P(_Comm), P(_Result)]
    lib.bdeg_degree_walk_sharded.restype = ctypes.c_int
    lib.bdeg_steal_create.argtypes = [ctypes.c_int32, ctypes.c_char_p]
    lib.bdeg_steal_create.restype = ctypes.c_int
    lib.bdeg_steal_attach.argtypes = [plan_t, ctypes.c_char_p]
    lib.bdeg_steal_attach.restype = ctypes.c_int
    lib.bdeg_rank_modp.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int64), ctypes.c_uint32,
                                   ctypes.c_int32, ctypes.c_void_p, P(ctypes.c_int64)]
    lib.bdeg_rank_modp.restype = ctypes.c_int
    lib.bdeg_dimension_modp.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int64), ctypes.c_int32,
                                        P(ctypes.c_int32)]
    lib.bdeg_dimension_modp.restype = ctypes.c_int
    lib.bdeg_smith_gpu.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int64), ctypes.c_int32,
                                   ctypes.c_void_p, P(ctypes.c_int64), P(ctypes.c_uint64), P(ctypes.c_uint64),
                                   P(ctypes.c_int64)]
    lib.bdeg_smith_gpu.restype = ctypes.c_int
    lib.bdeg_launch_count.argtypes = []
    lib.bdeg_launch_count.restype = ctypes.c_uint64
    for name in ["bdeg_plan", "bdeg_plan_points", "bdeg_plan_info", "bdeg_plan_points_get", "bdeg_set_workspace",
                 "bdeg_degree", "bdeg_degree_range", "bdeg_degree_partial", "bdeg_finalize",
                 "bdeg_relift"]:
        getattr(lib, name).restype = ctypes.c_int
    return lib


lib = _load()


def steal_create(device: int) -> bytes:
    """Rank 0: allocate the cross-GPU item counters, return their IPC handle."""
    buf = ctypes.create_string_buffer(64)
    _check(lib.bdeg_steal_create(device, buf))
    return buf.raw


def dimension_modp(A, device=None) -> int:
    """dim V*(x^A - b) = n - rank A by GPU row reduction mod 2 primes."""
    buf, n, m = _matrix_i64(A)
    d = ctypes.c_int32()
    _check(lib.bdeg_dimension_modp(n, m, buf, _current_device() if device is None else device, ctypes.byref(d)))
    return d.value


def smith_gpu(A, device=None):
    """Exact (rank, |prod d_j|, unit pivots) of A by GPU unit-pivot elimination
    plus the host Smith form of the residual (bdeg_smith_gpu)."""
    buf, n, m = _matrix_i64(A)
    r, lo, hi, piv = ctypes.c_int64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int64()
    _check(lib.bdeg_smith_gpu(n, m, buf, _current_device() if device is None else device, None,
                              ctypes.byref(r), ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(piv)))
    return r.value, (hi.value << 64) | lo.value, piv.value


def launch_count() -> int:
    return int(lib.bdeg_launch_count())


@dataclass
class Result:
    n: int
    rank: int
    dim: int
    K: int
    N: int
    tier: int
    homogeneous: bool
    inner_levels: int
    components: int
    degree: int
    candidates: int
    cells: int
    singular: int
    ties: int
    overflow_reruns: int
    updates: int
    leaves: int
    dead_leaves: int
    relifts: int
    consistent: bool
    singular_complete: bool
    seed_used: int
    total_candidates: int
    plan_ms: float
    kernel_ms: float
    total_ms: float
    wide_reruns: int = 0
    dead_full: bool = False
    extra: dict = field(default_factory=dict)


def _result(r: _Result) -> Result:
    deg = (r.deg_hi << 64) | r.deg_lo
    comps = (r.comp_hi << 64) | r.comp_lo
    return Result(n=r.n, rank=r.rank, dim=r.dim, K=r.K, N=r.N, tier=r.tier,
                  homogeneous=bool(r.homogeneous), inner_levels=r.inner_levels,
                  components=comps, degree=deg, candidates=r.candidates, cells=r.cells,
                  singular=r.singular, ties=r.ties, overflow_reruns=r.overflow_reruns,
                  updates=r.updates, leaves=r.leaves, dead_leaves=r.dead_leaves,
                  relifts=r.relifts,
                  consistent=bool(r.consistent), singular_complete=bool(r.singular_complete),
                  seed_used=r.seed_used,
                  total_candidates=r.total_candidates, plan_ms=r.plan_ms,
                  kernel_ms=r.kernel_ms, total_ms=r.total_ms, wide_reruns=r.wide_reruns,
                  dead_full=bool(r.dead_full))


def _current_device():
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # noqa: BLE001 - torch is plumbing only
        pass
    return 0


def _options(seed=1, lift_bits=20, max_relift=32, device=None, rank=0, world=1, stream=None,
             flags=0, inner_levels=-1, ctas_per_sm=0) -> _Options:
    if device is None:      # the caller's current CUDA device (one process per GPU)
        device = _current_device()
    o = _Options()
    lib.bdeg_default_options(ctypes.byref(o))
    o.seed = seed & ((1 << 64) - 1)
    o.lift_bits = lift_bits
    o.max_relift = max_relift
    o.device = device
    o.rank = rank
    o.world = world
    o.stream = stream
    o.flags = flags
    o.inner_levels = inner_levels
    o.ctas_per_sm = ctas_per_sm
    return o


def _i64(values):
    vals = [int(v) for v in values]
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)


def _matrix_i64(A):
    """Row-major int64 buffer of an n x m matrix (list of rows or a numpy array)."""
    try:
        import numpy as np
        arr = np.ascontiguousarray(np.asarray(A, dtype=np.int64))
        if arr.ndim == 2 and arr.size > 0:
            ptr = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            ptr._keep = arr                      # the array outlives the call through the pointer
            return ptr, arr.shape[0], arr.shape[1]
    except (ImportError, ValueError, OverflowError):
        pass
    n = len(A)
    m = len(A[0]) if n else 0
    return _i64([A[i][j] for i in range(n) for j in range(m)]), n, m


def _check(status, plan=None):
    if status != BDEG_OK:
        msg = lib.bdeg_last_error(plan).decode(errors="replace")
        raise BdegError(status, msg)


def _current_stream():
    try:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream).value
    except Exception:  # noqa: BLE001 - torch is plumbing only
        pass
    return None


class Plan:
    """A planned degree computation (one bdeg_plan_t)."""

    def __init__(self, handle, keep):
        self._h = handle
        self._keep = keep
        self._ws = None
        self._world = 1

    # -- construction ------------------------------------------------
    @classmethod
    def from_system(cls, A, b=None, lifting=None, **opts):
        """x^A = b with A given as n rows of m ints."""
        n = len(A)
        m = len(A[0]) if n else 0
        if "stream" not in opts:
            opts["stream"] = _current_stream()
        pr = _Problem()
        pr.n, pr.m = n, m
        Abuf = _i64([A[i][j] for i in range(n) for j in range(m)])
        pr.A = Abuf
        keep = [Abuf]
        if b is not None:
            bre = (ctypes.c_double * max(1, m))(*[complex(x).real for x in b])
            bim = (ctypes.c_double * max(1, m))(*[complex(x).imag for x in b])
            pr.b_re, pr.b_im = bre, bim
            keep += [bre, bim]
        if lifting is not None:
            if len(lifting) != n + 1:
                raise ValueError("lifting needs n+1 values (variables, then the origin)")
            lb = _i64(lifting)
            pr.lifting = lb
            keep.append(lb)
        o = _options(**opts)
        h = ctypes.c_void_p()
        _check(lib.bdeg_plan(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(h)))
        plan = cls(h, keep)
        plan._world = o.world
        return plan

    @classmethod
    def from_points(cls, V, lifting=None, **opts):
        """Lifted vector configuration: N K-vectors (point-major)."""
        N = len(V)
        K = len(V[0])
        if "stream" not in opts:
            opts["stream"] = _current_stream()
        Vb = _i64([x for v in V for x in v])
        lb = _i64(lifting) if lifting is not None else None
        o = _options(**opts)
        h = ctypes.c_void_p()
        _check(lib.bdeg_plan_points(K, N, Vb, lb, ctypes.byref(o), ctypes.byref(h)))
        plan = cls(h, [Vb, lb])
        plan._world = o.world
        return plan

    # -- queries -----------------------------------------------------
    def info(self) -> Result:
        r = _Result()
        _check(lib.bdeg_plan_info(self._h, ctypes.byref(r)), self._h)
        return _result(r)

    def points(self):
        """(K, V point-major as tuples, lifting) the plan enumerates (bdeg_plan_points_get)."""
        info = self.info()
        K, N = info.K, info.N
        Vb = (ctypes.c_int64 * max(1, K * N))()
        wb = (ctypes.c_int64 * max(1, N))()
        _check(lib.bdeg_plan_points_get(self._h, Vb, wb), self._h)
        V = [tuple(Vb[l * K + i] for i in range(K)) for l in range(N)]
        return K, V, [wb[l] for l in range(N)]

    def num_items(self) -> int:
        return int(lib.bdeg_num_items(self._h))

    def item_range(self, item: int):
        b, e = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.bdeg_item_range(self._h, item, ctypes.byref(b), ctypes.byref(e)), self._h)
        return b.value, e.value

    def queue_info(self):
        """dict(n_items, n_split, n_static, grab) of the work queue (bdeg_queue_info)."""
        v = [ctypes.c_uint64() for _ in range(4)]
        _check(lib.bdeg_queue_info(self._h, *[ctypes.byref(x) for x in v]), self._h)
        return dict(zip(("n_items", "n_split", "n_static", "grab"), (x.value for x in v)))

    def shard_items(self, rank: int, world: int):
        """Queue positions of `rank` under bdeg_degree_partial's static rule
        (no stealing counter attached): rank, rank + world, ..."""
        return list(range(rank, self.num_items(), world))

    def steal_attach(self, handle: bytes):
        """Take work items from the shared cross-GPU queue (bdeg_steal_attach)."""
        _check(lib.bdeg_steal_attach(self._h, handle), self._h)

    def workspace_bytes(self) -> int:
        return int(lib.bdeg_workspace_bytes(self._h))

    def use_torch_workspace(self, device=None):
        """Give the plan a torch-allocated device workspace (PyTorch memory)."""
        import torch
        nbytes = self.workspace_bytes()
        if nbytes == 0:
            return None
        dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        ptr = ws.data_ptr()
        aligned = (ptr + 255) & ~255
        _check(lib.bdeg_set_workspace(self._h, ctypes.c_void_p(aligned), nbytes), self._h)
        self._ws = ws
        return ws

    def degree(self) -> Result:
        r = _Result()
        _check(lib.bdeg_degree(self._h, ctypes.byref(r)), self._h)
        return _result(r)

    def degree_walk(self) -> Result:
        """Output-sensitive degree by walking the subdivision."""
        r = _Result()
        _check(lib.bdeg_degree_walk(self._h, ctypes.byref(r)), self._h)
        return _result(r)

    def degree_walk_sharded(self, allreduce_sum, alltoall_counts, alltoall_cells) -> Result:
        """The walk with its hash set sharded over the ranks (bdeg_degree_walk_sharded).
        The three callables implement the collectives (multi.degree_walk_distributed):
          allreduce_sum(list[int]) -> list[int];  alltoall_counts(list[int]) -> list[int];
          alltoall_cells(d_send_ptr, send_counts, d_recv_ptr, recv_counts) -> None."""
        errors = []

        def ar(_ctx, vals, n):
            try:
                out = allreduce_sum([vals[i] for i in range(n)])
                for i in range(n):
                    vals[i] = int(out[i])
                return 0
            except Exception as e:  # noqa: BLE001 - reported as BDEG_E_COMM
                errors.append(e)
                return 1

        def ac(_ctx, send, recv):
            try:
                w = self._world
                out = alltoall_counts([send[i] for i in range(w)])
                for i in range(w):
                    recv[i] = int(out[i])
                return 0
            except Exception as e:  # noqa: BLE001
                errors.append(e)
                return 1

        def ax(_ctx, d_send, scnt, d_recv, rcnt):
            try:
                w = self._world
                alltoall_cells(d_send or 0, [scnt[i] for i in range(w)], d_recv or 0, [rcnt[i] for i in range(w)])
                return 0
            except Exception as e:  # noqa: BLE001
                errors.append(e)
                return 1

        cbs = (_ALLREDUCE(ar), _A2A_COUNTS(ac), _A2A_CELLS(ax))
        comm = _Comm(None, *cbs)
        r = _Result()
        st = lib.bdeg_degree_walk_sharded(self._h, ctypes.byref(comm), ctypes.byref(r))
        if st != BDEG_OK and errors:
            raise BdegError(st, f"{lib.bdeg_last_error(self._h).decode(errors='replace')}: {errors[0]!r}")
        _check(st, self._h)
        return _result(r)

    def cells(self, begin: int = 0, end: int = None, capacity: int = 1 << 20):
        """Cells among ranks [begin, end) as a list of (point-index tuple, |det|)."""
        if end is None:
            end = self.info().total_candidates
        buf = (ctypes.c_uint64 * (2 * max(1, capacity)))()
        n = ctypes.c_uint64()
        _check(lib.bdeg_cells(self._h, begin, end, buf, capacity, ctypes.byref(n)), self._h)
        if n.value > capacity:
            raise BdegError(BDEG_E_TOO_LARGE, f"{n.value} cells exceed capacity {capacity}")
        out = []
        for i in range(n.value):
            m, v = buf[2 * i], buf[2 * i + 1]
            out.append((tuple(l for l in range(64) if (m >> l) & 1), v))
        return sorted(out)

    def cell_normal(self, cell):
        """Exact lifted hyperplane h = h_num/den of a cell (point-index tuple):
        h . v_c = omega_c on the cell (the paper's inner normal)."""
        from fractions import Fraction
        lo = sum(1 << l for l in cell if l < 64)
        hi = sum(1 << (l - 64) for l in cell if l >= 64)
        K = len(cell)
        num = (ctypes.c_int64 * K)()
        den = ctypes.c_int64()
        _check(lib.bdeg_cell_normal(self._h, lo, hi, num, ctypes.byref(den)), self._h)
        return [Fraction(num[i], den.value) for i in range(K)]

    def degree_range(self, begin: int, end: int) -> Result:
        r = _Result()
        _check(lib.bdeg_degree_range(self._h, begin, end, ctypes.byref(r)), self._h)
        return _result(r)

    def degree_partial(self, d_slots_ptr: int):
        """Enqueue this rank's shard into a device int64[16] buffer (pointer)."""
        _check(lib.bdeg_degree_partial(self._h, ctypes.c_void_p(d_slots_ptr)), self._h)

    def finalize(self, h_slots) -> Result:
        buf = _i64(h_slots)
        r = _Result()
        _check(lib.bdeg_finalize(self._h, buf, ctypes.byref(r)), self._h)
        return _result(r)

    def relift(self, attempt: int):
        _check(lib.bdeg_relift(self._h, attempt), self._h)

    def close(self):
        if self._h:
            lib.bdeg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def degree(A, b=None, lifting=None, **opts) -> Result:
    """deg of each component of V*(x^A - b) (Prop. 4) on the GPU."""
    with Plan.from_system(A, b, lifting, **opts) as p:
        return p.degree()


def degree_points(V, lifting=None, **opts) -> Result:
    with Plan.from_points(V, lifting, **opts) as p:
        return p.degree()
