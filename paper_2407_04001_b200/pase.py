"""Thin ctypes binding of libpase.so (include/pase.h).  Argument marshalling only: every
step of the search runs inside the library (host C++ + sm_100a kernels).  There is no
CPU fallback: if libpase.so is missing or no CUDA device is present, calls fail loudly.

The names mirror the C ABI: pase_create / pase_solve / pase_get_stats / ... plus a
convenience ``solve(graph, p, ...)``.  Graphs are the dicts of ``zoo.py``.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libpase.so")

PASE_MAX_DIMS = 8
PASE_MAX_HALO = 4
PASE_MAX_DEP = 12
PASE_HANDLE_BYTES = 256
TRACE_WORDS = 22
PASE_CFG_EXACT_P, PASE_CFG_LE_P = 0, 1
STATUS = {0: "PASE_OK", 1: "PASE_ERR_INVALID", 2: "PASE_ERR_RESOURCE", 3: "PASE_ERR_CUDA",
          4: "PASE_ERR_NCCL", 5: "PASE_ERR_STATE"}
POLICIES = {"exact_p": PASE_CFG_EXACT_P, "le_p": PASE_CFG_LE_P}
ORDERINGS = {"sortnodes": 0, "bfs": 1}


class pase_node(C.Structure):
    _fields_ = [
        ("n_dims", C.c_int32),
        ("size", C.c_int64 * PASE_MAX_DIMS),
        ("splittable_mask", C.c_uint32),
        ("n_out_axes", C.c_int32),
        ("out_axes", C.c_int32 * PASE_MAX_DIMS),
        ("n_w_axes", C.c_int32),
        ("w_axes", C.c_int32 * PASE_MAX_DIMS),
        ("flop_dims_mask", C.c_uint32),
        ("flops_per_point", C.c_int64),
        ("n_halo", C.c_int32),
        ("halo_spatial", C.c_int32 * PASE_MAX_HALO),
        ("halo_filter", C.c_int32 * PASE_MAX_HALO),
        ("elem_bytes", C.c_int32),
        ("n_in_axes", C.c_int32),
        ("in_axes", C.c_int32 * PASE_MAX_DIMS),
    ]


class pase_edge(C.Structure):
    _fields_ = [("src", C.c_int32), ("dst", C.c_int32), ("axis_map", C.c_int32 * PASE_MAX_DIMS)]


class pase_graph(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nodes", C.POINTER(pase_node)),
                ("n_edges", C.c_int32), ("edges", C.POINTER(pase_edge))]


class pase_machine(C.Structure):
    _fields_ = [
        ("flops_per_device", C.c_double),
        ("link_bandwidth", C.c_double),
        ("cfg_policy", C.c_int32),
        ("ordering", C.c_int32),
        ("table_budget_bytes", C.c_uint64),
        ("redundant_below_bytes", C.c_uint64),
        ("cuda_device", C.c_int32),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("virtual_ranks", C.c_int32),
        ("reserved", C.c_void_p),
        ("cuda_stream", C.c_void_p),
    ]


class pase_stats(C.Structure):
    _fields_ = [
        ("n_vertices", C.c_int32), ("n_edges", C.c_int32),
        ("max_dep", C.c_int32), ("max_configs", C.c_int32),
        ("tree_levels", C.c_int32), ("n_launches", C.c_int32),
        ("candidates", C.c_uint64), ("table_entries", C.c_uint64),
        ("cost_entries", C.c_uint64), ("alg_bytes_dp", C.c_uint64),
        ("alg_bytes_tables", C.c_uint64), ("comm_bytes", C.c_uint64),
        ("ms_create", C.c_double), ("ms_nccl_init", C.c_double),
        ("ms_solve", C.c_double), ("ms_tables", C.c_double), ("ms_dp", C.c_double),
        ("dp_fp64_ops", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
    ]


EXPORTS = ["pase_create", "pase_solve", "pase_get_stats", "pase_last_error", "pase_destroy",
           "pase_get_configs", "pase_get_order", "pase_get_cost_tables", "pase_get_dp_table",
           "pase_table_entries", "pase_set_cost_tables", "pase_set_profiling", "pase_get_trace",
           "pase_launch", "pase_finish", "pase_export_handle", "pase_connect", "pase_get_schedule",
           "pase_evaluate", "pase_brute_force", "pase_assign_devices"]

_lib = None


class PaseError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def load(path: str = SO):
    """Load libpase.so (no fallback: a missing library is an error).  PASE_LIB names an A/B
    build variant of it (tuning only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PASE_LIB", path)
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P = C.POINTER
    ctx_p = C.c_void_p
    L.pase_create.argtypes = [P(pase_graph), C.c_int32, P(pase_machine), P(ctx_p)]
    L.pase_solve.argtypes = [ctx_p, P(C.c_int32), P(C.c_int32), P(C.c_double)]
    L.pase_get_stats.argtypes = [ctx_p, P(pase_stats)]
    L.pase_last_error.argtypes = [ctx_p]
    L.pase_last_error.restype = C.c_char_p
    L.pase_destroy.argtypes = [ctx_p]
    L.pase_destroy.restype = None
    L.pase_get_configs.argtypes = [ctx_p, P(C.c_int32), P(C.c_int32)]
    L.pase_get_order.argtypes = [ctx_p, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32)]
    L.pase_get_cost_tables.argtypes = [ctx_p, C.c_int32, C.c_int32, P(C.c_double)]
    L.pase_get_dp_table.argtypes = [ctx_p, C.c_int32, P(C.c_double), P(C.c_uint16)]
    L.pase_table_entries.argtypes = [ctx_p, C.c_int32]
    L.pase_table_entries.restype = C.c_int64
    L.pase_set_cost_tables.argtypes = [ctx_p, P(C.c_double), P(C.c_double)]
    L.pase_set_profiling.argtypes = [ctx_p, C.c_int32]
    L.pase_get_trace.argtypes = [ctx_p, P(C.c_int64), C.c_int64]
    L.pase_get_trace.restype = C.c_int64
    L.pase_launch.argtypes = [ctx_p]
    L.pase_finish.argtypes = [ctx_p, P(C.c_int32), P(C.c_int32), P(C.c_double)]
    L.pase_export_handle.argtypes = [ctx_p, C.c_void_p]
    L.pase_connect.argtypes = [ctx_p, C.c_void_p]
    L.pase_get_schedule.argtypes = [ctx_p, P(C.c_int32), P(C.c_int64), P(C.c_int32)]
    L.pase_get_schedule.restype = C.c_int64
    L.pase_evaluate.argtypes = [ctx_p, P(C.c_int32), C.c_int64, P(C.c_double)]
    L.pase_brute_force.argtypes = [ctx_p, C.c_uint64, P(C.c_int32), P(C.c_double), P(C.c_uint64)]
    L.pase_assign_devices.argtypes = [ctx_p, P(C.c_int32), P(C.c_int32), P(C.c_double)]
    for f in ("pase_assign_devices", "pase_evaluate", "pase_brute_force", "pase_create", "pase_solve", "pase_get_stats", "pase_get_configs", "pase_get_order",
              "pase_get_cost_tables", "pase_get_dp_table", "pase_set_cost_tables", "pase_set_profiling",
              "pase_launch", "pase_finish", "pase_export_handle", "pase_connect"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def marshal_graph(graph: dict):
    """dict -> (pase_graph, keepalive).  Layout per include/pase.h; the node/edge arrays are
    numpy structured arrays with the ctypes structs' dtype, filled from one int64 matrix
    (one row of every integer field per node, one array conversion)."""
    nodes = graph["nodes"]
    edges = graph["edges"]
    n, m = len(nodes), len(edges)
    NA = np.zeros(max(n, 1), dtype=np.dtype(pase_node))
    D, HL = PASE_MAX_DIMS, PASE_MAX_HALO
    Z8, Z4 = [0] * D, [0] * HL
    rows = []
    for v, nd in enumerate(nodes):
        if nd["id"] != v:
            raise ValueError(f"node {v}: id {nd['id']} must equal its index")
        dims = nd["dims"]
        nd_ = len(dims)
        if nd_ > D:
            raise ValueError(f"node {v}: more than {D} dims")
        oa = nd["out_axes"]
        w = nd.get("w_axes") or []
        fd = nd.get("flop_dims")
        halo = nd.get("halo") or []
        ins = nd.get("in_axes") or []
        if len(halo) > HL:
            raise ValueError(f"node {v}: more than {HL} halo pairs")
        mask = 0
        sizes = []
        for k, d in enumerate(dims):
            sizes.append(d["size"])
            if d.get("splittable", True):
                mask |= 1 << k
        fmask = 0
        if fd is not None:
            for k in fd:
                fmask |= 1 << k
        rows.append([nd_, *sizes, *Z8[nd_:], mask, len(oa), *oa, *Z8[len(oa):], len(w), *w, *Z8[len(w):],
                     fmask, nd.get("flops_per_point", 2), len(halo), *[h for h, _ in halo], *Z4[len(halo):],
                     *[f for _, f in halo], *Z4[len(halo):], nd.get("elem_bytes", 4),
                     len(ins), *ins, *Z8[len(ins):]])
    if n:
        M = np.array(rows, dtype=np.int64)
        c = 0
        for k, width in (("n_dims", 1), ("size", D), ("splittable_mask", 1), ("n_out_axes", 1), ("out_axes", D),
                         ("n_w_axes", 1), ("w_axes", D), ("flop_dims_mask", 1), ("flops_per_point", 1),
                         ("n_halo", 1), ("halo_spatial", HL), ("halo_filter", HL), ("elem_bytes", 1),
                         ("n_in_axes", 1), ("in_axes", D)):
            NA[k] = M[:, c] if width == 1 else M[:, c:c + width]
            c += width
    EA = np.zeros(max(m, 1), dtype=np.dtype(pase_edge))
    if m:
        E = np.array([[ed["src"], ed["dst"], *ed["axis_map"], *[-1] * (D - len(ed["axis_map"]))] for ed in edges],
                     dtype=np.int64)
        EA["src"] = E[:, 0]
        EA["dst"] = E[:, 1]
        EA["axis_map"] = E[:, 2:]
    g = pase_graph(n, NA.ctypes.data_as(C.POINTER(pase_node)), m, EA.ctypes.data_as(C.POINTER(pase_edge)))
    return g, (NA, EA)


class Graph:
    """A graph already in the C ABI's input layout (pase_graph + node / edge arrays): marshal a
    dict once, then create any number of contexts from it (Context accepts a Graph or a dict)."""

    def __init__(self, graph: dict):
        self.graph = graph
        self.c_graph, self._keep = marshal_graph(graph)
        self.n_dims = [len(nd["dims"]) for nd in graph["nodes"]]


def make_machine(flops: float = 1e13, bandwidth: float = 1e10, policy: int = PASE_CFG_EXACT_P,
                 device: int = 0, stream: Optional[int] = None, rank: int = 0, world: int = 1,
                 virtual_ranks: bool = False, table_budget: int = 0,
                 redundant_below: int = 4 << 20, ordering: int = 0) -> pase_machine:
    m = pase_machine()
    m.flops_per_device, m.link_bandwidth = float(flops), float(bandwidth)
    m.cfg_policy = int(policy)
    m.ordering = int(ordering)
    m.table_budget_bytes = int(table_budget)
    m.redundant_below_bytes = int(redundant_below)
    m.cuda_device, m.rank, m.world = int(device), int(rank), int(world)
    m.virtual_ranks = 1 if virtual_ranks else 0
    m.cuda_stream = stream
    return m


class Context:
    """Owns one pase_ctx (pase_create ... pase_destroy)."""

    def __init__(self, graph, p: int, policy="exact_p", flops: Optional[float] = None,
                 bandwidth: Optional[float] = None, device: int = 0, stream: Optional[int] = None,
                 rank: int = 0, world: int = 1, virtual_ranks: bool = False, table_budget: int = 0,
                 redundant_below: int = 4 << 20, ordering="sortnodes"):
        L = load()
        G = graph if isinstance(graph, Graph) else None
        if G is not None:
            graph = G.graph
        mach_d = graph.get("machine") or {}
        flops = flops if flops is not None else mach_d.get("flops", 1e13)
        bandwidth = bandwidth if bandwidth is not None else mach_d.get("bandwidth", 1e10)
        pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
        if G is not None:
            g, self._keep = G.c_graph, G._keep
        else:
            g, self._keep = marshal_graph(graph)
        self.graph = graph
        self.n, self.m, self.p = len(graph["nodes"]), len(graph["edges"]), int(p)
        self._nd = G.n_dims if G is not None else [len(nd["dims"]) for nd in graph["nodes"]]
        order = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
        self._mach = make_machine(flops, bandwidth, pol, device, stream, rank, world, virtual_ranks,
                                  table_budget, redundant_below, order)
        self.rank, self.world = rank, world
        h = C.c_void_p()
        st = L.pase_create(C.byref(g), int(p), C.byref(self._mach), C.byref(h))
        if st != 0:
            raise PaseError(st, L.pase_last_error(None).decode())
        self._h = h
        self._L = L

    def _chk(self, st: int) -> None:
        if st != 0:
            raise PaseError(st, self._L.pase_last_error(self._h).decode())

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.pase_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- a5-a8
    def solve(self) -> Dict[str, object]:
        cfg = np.zeros((self.n, PASE_MAX_DIMS), np.int32)
        idx = np.zeros(self.n, np.int32)
        tot = C.c_double()
        self._chk(self._L.pase_solve(self._h, _ptr(cfg, C.c_int32), _ptr(idx, C.c_int32), C.byref(tot)))
        tuples = [tuple(r[:d]) for r, d in zip(cfg.tolist(), self._nd)]
        return {"cost": tot.value, "config_index": idx, "configs": tuples}

    # ---- row f2: Eq. 1 on the GPU
    def evaluate(self, config_index) -> np.ndarray:
        """pase_evaluate: Eq. 1 cost of each strategy (rows of config indices, one per node)."""
        a = np.ascontiguousarray(np.atleast_2d(np.asarray(config_index, dtype=np.int32)))
        if a.shape[1] != self.n:
            raise ValueError(f"strategies must have {self.n} entries, got {a.shape[1]}")
        out = np.zeros(a.shape[0], np.float64)
        self._chk(self._L.pase_evaluate(self._h, _ptr(a, C.c_int32), a.shape[0], _ptr(out, C.c_double)))
        return out

    def brute_force(self, max_strategies: int = 0) -> Dict[str, object]:
        """pase_brute_force: min of Eq. 1 over all prod K_v strategies (lowest index wins ties)."""
        idx = np.zeros(self.n, np.int32)
        tot = C.c_double()
        ns = C.c_uint64()
        self._chk(self._L.pase_brute_force(self._h, max_strategies, _ptr(idx, C.c_int32), C.byref(tot),
                                           C.byref(ns)))
        return {"cost": tot.value, "config_index": idx, "n_strategies": ns.value}

    # ---- row f3: device assignment
    def assign_devices(self, config_index):
        """pase_assign_devices: greedy placement of each vertex's shards on the p devices
        (P:288-294).  Returns (device int32[n, p] with -1 padding, realized t_x bytes[m])."""
        idx = np.ascontiguousarray(np.asarray(config_index, dtype=np.int32))
        dev = np.zeros((self.n, self.p), np.int32)
        tx = np.zeros(max(self.m, 1), np.float64)
        self._chk(self._L.pase_assign_devices(self._h, _ptr(idx, C.c_int32), _ptr(dev, C.c_int32),
                                              _ptr(tx, C.c_double)))
        return dev, tx[:self.m]

    def launch(self) -> None:
        """pase_launch: enqueue one solve (a multi-GPU group launches every rank first)."""
        self._chk(self._L.pase_launch(self._h))

    def finish(self) -> Dict[str, object]:
        """pase_finish: wait for the launched solve; same result as solve()."""
        cfg = np.zeros((self.n, PASE_MAX_DIMS), np.int32)
        idx = np.zeros(self.n, np.int32)
        tot = C.c_double()
        self._chk(self._L.pase_finish(self._h, _ptr(cfg, C.c_int32), _ptr(idx, C.c_int32), C.byref(tot)))
        tuples = [tuple(r[:d]) for r, d in zip(cfg.tolist(), self._nd)]
        return {"cost": tot.value, "config_index": idx, "configs": tuples}

    def export_handle(self) -> bytes:
        buf = C.create_string_buffer(PASE_HANDLE_BYTES)
        self._chk(self._L.pase_export_handle(self._h, buf))
        return buf.raw

    def connect(self, handles: Sequence[bytes]) -> None:
        """pase_connect with the group's handles ordered by rank."""
        blob = b"".join(handles)
        buf = C.create_string_buffer(blob, len(blob))
        self._chk(self._L.pase_connect(self._h, buf))

    def schedule(self) -> Dict[str, np.ndarray]:
        """pase_get_schedule: per-vertex (part, bcast, ntasks, pending, shape, glog, wlog, q2),
        tasks (vertex, first item, end item, kind: > 0 = wave-tail lane groups 2^kind), claim order."""
        nt = self._L.pase_get_schedule(self._h, None, None, None)
        vinfo = np.zeros((self.n, 8), np.int32)
        tasks = np.zeros((max(nt, 1), 4), np.int64)
        order = np.zeros(max(nt, 1), np.int32)
        self._L.pase_get_schedule(self._h, _ptr(vinfo, C.c_int32), _ptr(tasks, C.c_int64), _ptr(order, C.c_int32))
        return {"vinfo": vinfo, "tasks": tasks[:nt], "order": order[:nt]}

    def stats(self) -> Dict[str, float]:
        s = pase_stats()
        self._chk(self._L.pase_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in pase_stats._fields_}

    # ---- introspection
    def configs(self) -> List[np.ndarray]:
        K = np.zeros(self.n, np.int32)
        self._chk(self._L.pase_get_configs(self._h, _ptr(K, C.c_int32), None))
        T = np.zeros((int(K.sum()), PASE_MAX_DIMS), np.int32)
        self._chk(self._L.pase_get_configs(self._h, _ptr(K, C.c_int32), _ptr(T, C.c_int32)))
        out, off = [], 0
        for v in range(self.n):
            d = len(self.graph["nodes"][v]["dims"])
            out.append(T[off:off + K[v], :d].copy())
            off += K[v]
        return out

    def K(self) -> np.ndarray:
        K = np.zeros(self.n, np.int32)
        self._chk(self._L.pase_get_configs(self._h, _ptr(K, C.c_int32), None))
        return K

    def order(self):
        n = self.n
        sigma = np.zeros(n, np.int32)
        off = np.zeros(n + 1, np.int32)
        ids = np.zeros(n * PASE_MAX_DEP + 1, np.int32)
        par = np.zeros(n, np.int32)
        self._chk(self._L.pase_get_order(self._h, _ptr(sigma, C.c_int32), _ptr(off, C.c_int32),
                                         _ptr(ids, C.c_int32), _ptr(par, C.c_int32)))
        return sigma, [ids[off[i]:off[i + 1]].tolist() for i in range(n)], par

    def cost_tables(self):
        K = self.K()
        Ls = []
        for v in range(self.n):
            out = np.zeros(int(K[v]), np.float64)
            self._chk(self._L.pase_get_cost_tables(self._h, v, 0, _ptr(out, C.c_double)))
            Ls.append(out)
        Ws = []
        for e, ed in enumerate(self.graph["edges"]):
            out = np.zeros((int(K[ed["src"]]), int(K[ed["dst"]])), np.float64)
            self._chk(self._L.pase_get_cost_tables(self._h, e, 1, _ptr(out, C.c_double)))
            Ws.append(out)
        return Ls, Ws

    def dp_table(self, rank: int):
        n = self._L.pase_table_entries(self._h, rank)
        T = np.zeros(n, np.float64)
        A = np.zeros(n, np.uint16)
        self._chk(self._L.pase_get_dp_table(self._h, rank, _ptr(T, C.c_double), _ptr(A, C.c_uint16)))
        return T, A

    def trace(self) -> np.ndarray:
        """PASE_TRACE=1 timeline of the last solve, one row per DP task (ns, %globaltimer):
        (rank, smid, t_claim, t_start, t_computed, t_synced, t_end, then per warp 0..7
        t_gate_seen, t_gate_fenced (0: no gate))."""
        n = self._L.pase_get_trace(self._h, None, 0)
        if n <= 0:
            return np.zeros((0, TRACE_WORDS + 1), np.int64)
        buf = np.zeros(TRACE_WORDS * n, np.int64)
        self._L.pase_get_trace(self._h, _ptr(buf, C.c_int64), n)
        r = buf.reshape(n, TRACE_WORDS)
        out = np.zeros((n, TRACE_WORDS + 1), np.int64)
        out[:, 0] = r[:, 0] & 0xffffffff
        out[:, 1] = r[:, 0] >> 32
        out[:, 2:] = r[:, 1:]
        return out

    def set_cost_tables(self, Ls: Sequence[np.ndarray], Ws: Sequence[np.ndarray]) -> None:
        L = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64).ravel() for x in Ls]))
        W = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64).ravel() for x in Ws])
                                 if len(Ws) else np.zeros(1))
        self._chk(self._L.pase_set_cost_tables(self._h, _ptr(L, C.c_double), _ptr(W, C.c_double)))


def virtual_group(graph: dict, p: int, world: int, device: int = 0, **kw) -> List[Context]:
    """A multi-GPU group of `world` ranks sharing one device in this process (testing the
    partitioned path on a single GPU): create, export, connect."""
    import torch
    ctxs = []
    for r in range(world):
        st = torch.cuda.Stream(device=device)
        ctxs.append(Context(graph, p, device=device, rank=r, world=world, virtual_ranks=True,
                            stream=st.cuda_stream, **kw))
        ctxs[-1]._torch_stream = st
    handles = [c.export_handle() for c in ctxs]
    for c in ctxs:
        c.connect(handles)
    return ctxs


def solve_group(ctxs: Sequence[Context]) -> List[Dict[str, object]]:
    """Launch every rank of a (virtual) group, then wait for all."""
    for c in ctxs:
        c.launch()
    return [c.finish() for c in ctxs]


# C-ABI-named wrappers (same names as include/pase.h)
def pase_create(graph: dict, p: int, **kw) -> Context:
    return Context(graph, p, **kw)


def pase_solve(ctx: Context) -> Dict[str, object]:
    return ctx.solve()


def pase_get_stats(ctx: Context) -> Dict[str, float]:
    return ctx.stats()


def pase_destroy(ctx: Context) -> None:
    ctx.close()


def solve(graph: dict, p: int, policy="exact_p", **kw) -> Dict[str, object]:
    """One-shot search: create, solve, destroy.  Returns cost, configs, stats."""
    with Context(graph, p, policy=policy, **kw) as ctx:
        r = ctx.solve()
        r["stats"] = ctx.stats()
        return r
