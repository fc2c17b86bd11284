"""Thin ctypes binding of libsg2v.so (include/sg2v.h) — argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; PyTorch is
used only for device memory (the workspace), the current CUDA stream and
process groups.  There is no CPU fallback: if libsg2v.so is missing or no
B200 is visible, calls raise.

Names follow the C ABI: graph_load_csr, template_build, count, colorize,
workspace_bytes, plan_describe, profile_enable / profile_read.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from .build import LIB

OK, EINVAL, ENOTTREE, ENOMEM, ECUDA, ENCCL, EOVERFLOW = range(7)
F32, F64, U64 = 0, 1, 2
PRECISIONS = {"f32": F32, "f64": F64, "u64": U64}
GRAPH_VALIDATE, GRAPH_DEVICE_PTRS = 1, 2
_NAMES = {1: "EINVAL", 2: "ENOTTREE", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "EOVERFLOW"}


class Sg2vError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class Options(ctypes.Structure):
    _fields_ = [
        ("precision", ctypes.c_int),
        ("iter_offset", ctypes.c_int64),
        ("iter_stride", ctypes.c_int64),
        ("mode", ctypes.c_int32),
        ("nccl_comm", ctypes.c_void_p),
        ("device", ctypes.c_int32),
        ("mem_budget_bytes", ctypes.c_uint64),
        ("col_tile", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_uint64),
        ("row_values", ctypes.c_void_p),
        ("layout", ctypes.c_int32),
    ]


_lib = None
SYMBOLS = ["sg2v_graph_load_csr", "sg2v_graph_free", "sg2v_template_build", "sg2v_template_free",
           "sg2v_template_info", "sg2v_options_default", "sg2v_set_options", "sg2v_workspace_bytes",
           "sg2v_count", "sg2v_count_ex", "sg2v_colorize", "sg2v_plan_describe", "sg2v_plan_describe_n", "sg2v_profile_enable",
           "sg2v_profile_read", "sg2v_last_error", "sg2v_version", "sg2v_count_batch",
           "sg2v_workspace_bytes_batch", "sg2v_comm_unique_id", "sg2v_comm_init_nccl", "sg2v_comm_init_callback",
           "sg2v_comm_free", "sg2v_graph_load_partition", "sg2v_estimate",
           "sg2v_profile_read_launches", "sg2v_partition_relabel", "sg2v_graph_set_vertex_ids",
           "sg2v_profile_kernel_count"]

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p)


def lib():
    """dlopen libsg2v.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        lib = os.environ.get("SG2V_LIB", LIB)  # A/B experiments against another build of the library
        if not os.path.exists(lib):
            raise RuntimeError(f"{lib} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(lib)
        vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        P = ctypes.POINTER
        L.sg2v_graph_load_csr.argtypes = [i64, vp, vp, i64, ctypes.c_uint32, P(vp)]
        L.sg2v_graph_free.argtypes = [vp]
        L.sg2v_graph_free.restype = None
        L.sg2v_template_build.argtypes = [i32, vp, i32, P(vp)]
        L.sg2v_template_free.argtypes = [vp]
        L.sg2v_template_free.restype = None
        L.sg2v_template_info.argtypes = [vp, P(i32), P(ctypes.c_double), P(ctypes.c_double)]
        L.sg2v_options_default.argtypes = [P(Options)]
        L.sg2v_options_default.restype = None
        L.sg2v_set_options.argtypes = [P(Options)]
        L.sg2v_workspace_bytes.argtypes = [vp, vp, ctypes.c_int, P(u64)]
        L.sg2v_count.argtypes = [vp, vp, i32, i64, u64, vp, vp, vp]
        L.sg2v_count_ex.argtypes = [vp, vp, i32, i64, u64, P(Options), vp, vp, vp]
        L.sg2v_colorize.argtypes = [u64, i64, i64, i32, vp, vp]
        L.sg2v_count_batch.argtypes = [vp, vp, i32, i32, i64, u64, P(Options), vp, vp, vp]
        L.sg2v_comm_unique_id.argtypes = [vp]
        L.sg2v_comm_init_nccl.argtypes = [vp, i32, i32, P(vp)]
        L.sg2v_comm_init_callback.argtypes = [i32, i32, ALLGATHER_FN, vp, P(vp)]
        L.sg2v_comm_free.argtypes = [vp]
        L.sg2v_comm_free.restype = None
        L.sg2v_graph_load_partition.argtypes = [i64, i64, i64, vp, vp, i64, ctypes.c_uint32, P(vp)]
        L.sg2v_workspace_bytes_batch.argtypes = [vp, vp, i32, ctypes.c_int, P(u64)]
        L.sg2v_plan_describe.argtypes = [vp, vp, ctypes.c_int, vp, u64, P(u64)]
        L.sg2v_plan_describe_n.argtypes = [i64, i64, vp, ctypes.c_int, vp, u64, P(u64)]
        L.sg2v_estimate.argtypes = [vp, i64, vp, P(ctypes.c_double)]
        L.sg2v_profile_read_launches.argtypes = [i64, vp, vp, vp, vp, vp, P(i64)]
        L.sg2v_partition_relabel.argtypes = [i64, vp, vp, i32, vp, vp, vp]
        L.sg2v_graph_set_vertex_ids.argtypes = [vp, vp, i64]
        L.sg2v_profile_enable.argtypes = [i32]
        L.sg2v_profile_read.argtypes = [vp, vp, vp]
        L.sg2v_profile_kernel_count.argtypes = [P(u64)]
        L.sg2v_last_error.restype = ctypes.c_char_p
        L.sg2v_version.restype = ctypes.c_char_p
        for name in ("sg2v_graph_load_csr", "sg2v_template_build", "sg2v_template_info", "sg2v_set_options",
                     "sg2v_workspace_bytes", "sg2v_count", "sg2v_count_ex", "sg2v_colorize",
                     "sg2v_plan_describe", "sg2v_plan_describe_n", "sg2v_profile_enable", "sg2v_profile_read",
                     "sg2v_count_batch", "sg2v_workspace_bytes_batch", "sg2v_comm_unique_id",
                     "sg2v_comm_init_nccl", "sg2v_comm_init_callback", "sg2v_graph_load_partition",
                     "sg2v_estimate", "sg2v_profile_read_launches", "sg2v_partition_relabel",
                     "sg2v_graph_set_vertex_ids", "sg2v_profile_kernel_count"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != OK:
        raise Sg2vError(rc, lib().sg2v_last_error().decode())


def _torch():
    import torch
    return torch


def _cur_stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Graph:
    """Device CSR handle (sg2v_graph_load_csr)."""

    def __init__(self, handle, n, nnz):
        self._h = handle
        self.n = n
        self.nnz = nnz

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib().sg2v_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Template:
    """Validated tree template (sg2v_template_build)."""

    def __init__(self, handle, k, edges):
        self._h = handle
        self.k = k
        self.edges = edges

    @property
    def handle(self):
        return self._h

    def info(self):
        k = ctypes.c_int32()
        a = ctypes.c_double()
        p = ctypes.c_double()
        _check(lib().sg2v_template_info(self._h, ctypes.byref(k), ctypes.byref(a), ctypes.byref(p)))
        return {"k": k.value, "alpha": a.value, "P": p.value}

    def free(self):
        if self._h:
            lib().sg2v_template_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _set_stream_option(stream):
    o = Options()
    lib().sg2v_options_default(ctypes.byref(o))
    o.stream = stream if stream is not None else _cur_stream()
    return o


def graph_load_csr(n, row_offsets, col_indices, validate=False, stream=None) -> Graph:
    """row_offsets/col_indices: numpy arrays (host) or CUDA torch tensors (device)."""
    flags = GRAPH_VALIDATE if validate else 0
    if hasattr(row_offsets, "is_cuda") and row_offsets.is_cuda:
        torch = _torch()
        ro = row_offsets.to(torch.int64).contiguous()
        ci = col_indices.to(torch.int32).contiguous()
        flags |= GRAPH_DEVICE_PTRS
        p_ro, p_ci, nnz = ro.data_ptr(), ci.data_ptr() if ci.numel() else None, ci.numel()
        keep = (ro, ci)
    else:
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(col_indices, dtype=np.int32)
        p_ro = ro.ctypes.data
        p_ci = ci.ctypes.data if ci.size else None
        nnz = ci.size
        keep = (ro, ci)
    o = _set_stream_option(stream)
    _check(lib().sg2v_set_options(ctypes.byref(o)))
    h = ctypes.c_void_p()
    _check(lib().sg2v_graph_load_csr(int(n), p_ro, p_ci, int(nnz), flags, ctypes.byref(h)))
    del keep
    return Graph(h, int(n), int(nnz))


def template_build(k, edges, root_hint=-1) -> Template:
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1)) if len(edges) else None
    h = ctypes.c_void_p()
    _check(lib().sg2v_template_build(int(k), e.ctypes.data if e is not None else None, int(root_hint),
                                     ctypes.byref(h)))
    return Template(h, int(k), list(edges))


LAYOUTS = {"anchored": 0, "dense": 1, "anchored_plain": 2, "anchored_proj": 3}


def _set_layout(layout, mem_budget_bytes=0):
    """Thread-local options carry the layout and budget used by the planning queries."""
    o = Options()
    lib().sg2v_options_default(ctypes.byref(o))
    o.layout = LAYOUTS[layout]
    o.mem_budget_bytes = int(mem_budget_bytes)
    _check(lib().sg2v_set_options(ctypes.byref(o)))


def workspace_bytes(graph: Graph, tmpl: Template, precision="f32", layout="anchored", mem_budget_bytes=0) -> int:
    _set_layout(layout, mem_budget_bytes)
    b = ctypes.c_uint64()
    _check(lib().sg2v_workspace_bytes(graph.handle, tmpl.handle, PRECISIONS[precision], ctypes.byref(b)))
    return int(b.value)


def plan_describe(graph: Graph, tmpl: Template, precision="f32", layout="anchored", mem_budget_bytes=0) -> dict:
    _set_layout(layout, mem_budget_bytes)
    need = ctypes.c_uint64()
    _check(lib().sg2v_plan_describe(graph.handle, tmpl.handle, PRECISIONS[precision], None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(int(need.value))
    _check(lib().sg2v_plan_describe(graph.handle, tmpl.handle, PRECISIONS[precision], buf, need.value,
                                    ctypes.byref(need)))
    return json.loads(buf.value.decode())


def plan_describe_n(n: int, nnz: int, tmpl: Template, precision="f32", layout="anchored",
                    mem_budget_bytes=0) -> dict:
    """Host-only planning (no graph handle, no GPU)."""
    _set_layout(layout, mem_budget_bytes)
    need = ctypes.c_uint64()
    _check(lib().sg2v_plan_describe_n(int(n), int(nnz), tmpl.handle, PRECISIONS[precision], None, 0,
                                      ctypes.byref(need)))
    buf = ctypes.create_string_buffer(int(need.value))
    _check(lib().sg2v_plan_describe_n(int(n), int(nnz), tmpl.handle, PRECISIONS[precision], buf, need.value,
                                      ctypes.byref(need)))
    return json.loads(buf.value.decode())


class Workspace:
    """Device workspace allocated by torch and lent to the library."""

    def __init__(self, nbytes, device=None):
        torch = _torch()
        self.tensor = torch.empty(max(int(nbytes), 1), dtype=torch.uint8,
                                  device=device if device is not None else "cuda")
        self.nbytes = int(nbytes)

    @property
    def ptr(self):
        return self.tensor.data_ptr()


def count(graph: Graph, tmpl: Template, n_iter: int, seed: int, precision="f32", iter_offset=0,
          iter_stride=1, workspace: Workspace | None = None, stream=None, row_values=None,
          allow_overflow=False, mem_budget_bytes=0, layout="anchored", comm=None, col_tile=0):
    """sg2v_count_ex.  Returns (estimate, colorful) — colorful is float64[n_iter]
    (F32/F64) or uint64[n_iter] (U64, residues mod 2^64).  row_values: optional
    CUDA tensor (float64 or int64/uint64, n entries) receiving the per-vertex
    values of the last colouring.  layout: "anchored" (default) or "dense".
    comm: a Comm -> vertex-partitioned mode (graph from graph_load_partition)."""
    prec = PRECISIONS[precision]
    if workspace is None and graph.n > 0 and tmpl.k > 1 and comm is None:
        workspace = Workspace(workspace_bytes(graph, tmpl, precision, layout, mem_budget_bytes))
    o = Options()
    lib().sg2v_options_default(ctypes.byref(o))
    o.precision = prec
    o.iter_offset = int(iter_offset)
    o.iter_stride = int(iter_stride)
    o.stream = stream if stream is not None else _cur_stream()
    o.mem_budget_bytes = int(mem_budget_bytes)
    o.layout = LAYOUTS[layout]
    if comm is not None:
        o.mode = 1
        o.nccl_comm = comm.handle
        o.col_tile = int(col_tile)
    if workspace is not None:
        o.workspace = workspace.ptr
        o.workspace_bytes = workspace.nbytes
    if row_values is not None:
        o.row_values = row_values.data_ptr()
    est = ctypes.c_double()
    if prec == U64:
        out = np.zeros(n_iter, dtype=np.uint64)
        rc = lib().sg2v_count_ex(graph.handle, tmpl.handle, tmpl.k, int(n_iter), int(seed) & (2**64 - 1),
                                 ctypes.byref(o), ctypes.byref(est), None, out.ctypes.data)
    else:
        out = np.zeros(n_iter, dtype=np.float64)
        rc = lib().sg2v_count_ex(graph.handle, tmpl.handle, tmpl.k, int(n_iter), int(seed) & (2**64 - 1),
                                 ctypes.byref(o), ctypes.byref(est), out.ctypes.data, None)
    global LAST_STATUS
    LAST_STATUS = rc
    if rc == EOVERFLOW and allow_overflow:
        return est.value, out
    _check(rc)
    return est.value, out


LAST_STATUS = OK  # status of the last count() / count_batch() (EOVERFLOW with allow_overflow=True)


def estimate(tmpl: Template, colorful) -> float:
    """sg2v_estimate: mean/(P·α) of host per-colouring counts (replica shards)."""
    c = np.ascontiguousarray(colorful, dtype=np.float64)
    est = ctypes.c_double()
    rc = lib().sg2v_estimate(tmpl.handle, int(c.size), c.ctypes.data, ctypes.byref(est))
    if rc != EOVERFLOW:
        _check(rc)
    return est.value


def _handles(tmpls):
    arr = (ctypes.c_void_p * len(tmpls))(*[t.handle for t in tmpls])
    return arr


def workspace_bytes_batch(graph: Graph, tmpls, precision="f32", layout="anchored", mem_budget_bytes=0) -> int:
    _set_layout(layout, mem_budget_bytes)
    b = ctypes.c_uint64()
    _check(lib().sg2v_workspace_bytes_batch(graph.handle, _handles(tmpls), len(tmpls), PRECISIONS[precision],
                                            ctypes.byref(b)))
    return int(b.value)


def count_batch(graph: Graph, tmpls, n_iter: int, seed: int, precision="f32", iter_offset=0, iter_stride=1,
                workspace: Workspace | None = None, stream=None, allow_overflow=False, mem_budget_bytes=0,
                layout="anchored"):
    """sg2v_count_batch: m same-size templates on the same colourings.
    Returns (estimates[m], colorful[m, n_iter])."""
    m = len(tmpls)
    k = tmpls[0].k
    prec = PRECISIONS[precision]
    if workspace is None and graph.n > 0 and k > 1:
        workspace = Workspace(workspace_bytes_batch(graph, tmpls, precision, layout, mem_budget_bytes))
    o = Options()
    lib().sg2v_options_default(ctypes.byref(o))
    o.precision = prec
    o.iter_offset = int(iter_offset)
    o.iter_stride = int(iter_stride)
    o.stream = stream if stream is not None else _cur_stream()
    o.mem_budget_bytes = int(mem_budget_bytes)
    o.layout = LAYOUTS[layout]
    if workspace is not None:
        o.workspace = workspace.ptr
        o.workspace_bytes = workspace.nbytes
    est = np.zeros(m, dtype=np.float64)
    hs = _handles(tmpls)
    if prec == U64:
        out = np.zeros((m, n_iter), dtype=np.uint64)
        rc = lib().sg2v_count_batch(graph.handle, hs, m, k, int(n_iter), int(seed) & (2**64 - 1), ctypes.byref(o),
                                    est.ctypes.data, None, out.ctypes.data)
    else:
        out = np.zeros((m, n_iter), dtype=np.float64)
        rc = lib().sg2v_count_batch(graph.handle, hs, m, k, int(n_iter), int(seed) & (2**64 - 1), ctypes.byref(o),
                                    est.ctypes.data, out.ctypes.data, None)
    if rc == EOVERFLOW and allow_overflow:
        return est, out
    _check(rc)
    return est, out


class Comm:
    """sg2v_comm: NCCL (Comm.nccl) or host-callback (Comm.callback) transport."""

    def __init__(self, handle, rank, world, keep=None):
        self._h = handle
        self.rank = rank
        self.world = world
        self._keep = keep

    @property
    def handle(self):
        return self._h

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().sg2v_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, rank: int, world: int):
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        h = ctypes.c_void_p()
        _check(lib().sg2v_comm_init_nccl(buf, int(rank), int(world), ctypes.byref(h)))
        return cls(h, rank, world)

    @classmethod
    def callback(cls, rank: int, world: int, allgather):
        """allgather(send: bytes) -> bytes of world*len(send) (rank-major)."""
        def _fn(send, recv, nbytes, user):
            try:
                data = ctypes.string_at(send, nbytes)
                out = allgather(data)
                ctypes.memmove(recv, out, len(out))
                return 0
            except Exception:
                return 1
        cfn = ALLGATHER_FN(_fn)
        h = ctypes.c_void_p()
        _check(lib().sg2v_comm_init_callback(int(rank), int(world), cfn, None, ctypes.byref(h)))
        return cls(h, rank, world, keep=cfn)

    def free(self):
        if self._h:
            lib().sg2v_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def partition_rows(n_global: int, rank: int, world: int):
    """Rows of `rank` in the vertex-partitioned mode: [r*nl, r*nl + n_local)."""
    nl = (n_global + world - 1) // world
    begin = min(rank * nl, n_global)
    return begin, max(0, min(nl, n_global - begin))


def partition_relabel(row_offsets, col_indices, world):
    """sg2v_partition_relabel: (old_of_new, relabelled row_offsets, col_indices)."""
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(col_indices, dtype=np.int32)
    n = ro.size - 1
    oon = np.empty(max(n, 1), np.int32)
    ro2 = np.empty(n + 1, np.int64)
    ci2 = np.empty(max(ci.size, 1), np.int32)
    _check(lib().sg2v_partition_relabel(n, ro.ctypes.data, ci.ctypes.data if ci.size else None, int(world),
                                        oon.ctypes.data, ro2.ctypes.data, ci2.ctypes.data))
    return oon[:n], ro2, ci2[:ci.size]


def graph_set_vertex_ids(graph: Graph, orig_ids) -> None:
    ids = np.ascontiguousarray(orig_ids, dtype=np.int32)
    _check(lib().sg2v_graph_set_vertex_ids(graph.handle, ids.ctypes.data if ids.size else None, int(ids.size)))


def graph_load_partition(n_global, row_begin, n_local, row_offsets, col_indices, stream=None) -> Graph:
    """Local rows [row_begin, row_begin+n_local) (host numpy): row_offsets start at 0, global column ids."""
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(col_indices, dtype=np.int32)
    o = _set_stream_option(stream)
    _check(lib().sg2v_set_options(ctypes.byref(o)))
    h = ctypes.c_void_p()
    _check(lib().sg2v_graph_load_partition(int(n_global), int(row_begin), int(n_local), ro.ctypes.data,
                                           ci.ctypes.data if ci.size else None, int(ci.size), 0, ctypes.byref(h)))
    return Graph(h, int(n_local), int(ci.size))


def colorize(seed, j, n, k, out, stream=None):
    """K-COLOR into a CUDA uint8 tensor `out` (n entries)."""
    s = stream if stream is not None else _cur_stream()
    _check(lib().sg2v_colorize(int(seed) & (2**64 - 1), int(j), int(n), int(k), out.data_ptr(), s))


def profile_enable(on=True):
    _check(lib().sg2v_profile_enable(1 if on else 0))


KERNEL_CLASSES = ["color", "hist", "step", "top", "reduce"]


def profile_read():
    launches = np.zeros(5, np.int64)
    ms = np.zeros(5, np.float64)
    by = np.zeros(5, np.float64)
    _check(lib().sg2v_profile_read(launches.ctypes.data, ms.ctypes.data, by.ctypes.data))
    return {c: {"launches": int(launches[i]), "ms": float(ms[i]), "bytes": float(by[i])}
            for i, c in enumerate(KERNEL_CLASSES)}


def profile_read_launches():
    """Per-launch records: list of dicts {cls, ms, alg_bytes, impl_bytes, ema_terms}."""
    n = ctypes.c_int64()
    _check(lib().sg2v_profile_read_launches(0, None, None, None, None, None, ctypes.byref(n)))
    m = int(n.value)
    cls = np.zeros(max(m, 1), np.int32)
    ms, ab, ib, te = (np.zeros(max(m, 1), np.float64) for _ in range(4))
    _check(lib().sg2v_profile_read_launches(m, cls.ctypes.data, ms.ctypes.data, ab.ctypes.data, ib.ctypes.data,
                                            te.ctypes.data, ctypes.byref(n)))
    return [{"cls": KERNEL_CLASSES[int(cls[q])], "ms": float(ms[q]), "alg_bytes": float(ab[q]),
             "impl_bytes": float(ib[q]), "ema_terms": float(te[q])} for q in range(m)]


def profile_kernel_count() -> int:
    """Kernels of libsg2v launched since profile_enable(True) (every launch site counted)."""
    n = ctypes.c_uint64()
    _check(lib().sg2v_profile_kernel_count(ctypes.byref(n)))
    return int(n.value)


def version() -> str:
    return lib().sg2v_version().decode()
