"""ctypes wrapper of the plain CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module,
and this module never imports the product package (graphs arrive as plain dicts from
the shared input generators in paper_2407_04001_b200/zoo.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
MAXD, NODE_REC, EDGE_REC = 8, 49, 10
EXACT_P, LE_P = 0, 1


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", src, "-o", SO, "-lm"])
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(SO)
        P = C.POINTER
        i64p, i32p, f64p, u8p = P(C.c_int64), P(C.c_int32), P(C.c_double), P(C.c_uint8)
        sig = {
            "or_validate": [C.c_int, i64p, C.c_int, i64p],
            "or_configs": [C.c_int, i64p, C.c_int, C.c_int, i32p, i32p],
            "or_cost_tables": [C.c_int, i64p, C.c_int, i64p, C.c_int, C.c_int, C.c_double, C.c_double, f64p, f64p],
            "or_sortnodes": [C.c_int, C.c_int, i64p, i32p, i32p, i32p],
            "or_bfs_order": [C.c_int, C.c_int, i64p, i32p],
            "or_sets": [C.c_int, C.c_int, i64p, i32p, C.c_int, u8p, u8p, u8p, i32p, i32p],
            "or_table_sizes": [C.c_int, C.c_int, i64p, i32p, C.c_int, i64p, i64p],
            "or_dp": [C.c_int, C.c_int, i64p, i32p, f64p, f64p, C.c_int, C.c_int, C.c_int64, i32p, f64p, f64p, i32p],
            "or_dp_select": [C.c_int, C.c_int, i64p, i32p, f64p, f64p, C.c_int, C.c_int, i32p, f64p, C.c_int,
                             i32p, f64p, i32p],
            "or_dp_bfs_eq2": [C.c_int, C.c_int, i64p, i32p, f64p, f64p, C.c_int64, i32p, f64p],
            "or_brute": [C.c_int, C.c_int, i64p, i32p, f64p, f64p, C.c_int64, i32p, f64p],
            "or_assign": [C.c_int, i64p, C.c_int, i64p, C.c_int, i32p, i32p, f64p],
        }
        for name, args in sig.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int
        L.or_eval.argtypes = [C.c_int, C.c_int, i64p, i32p, f64p, f64p, i32p]
        L.or_eval.restype = C.c_double
        L.or_sum_h.argtypes = [C.c_int, C.c_int, i64p, i32p, f64p, f64p, i32p, i32p]
        L.or_sum_h.restype = C.c_double
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def encode(graph: dict) -> Tuple[np.ndarray, np.ndarray]:
    """Graph dict -> (node records int64[n, 49], edge records int64[m, 10])."""
    nodes = graph["nodes"]
    N = np.zeros((len(nodes), NODE_REC), dtype=np.int64)
    for v, nd in enumerate(nodes):
        assert nd["id"] == v
        r = N[v]
        dims = nd["dims"]
        r[0] = len(dims)
        for k, dd in enumerate(dims):
            r[1 + k] = dd["size"]
            if dd.get("splittable", True):
                r[9] |= 1 << k
        r[10] = len(nd["out_axes"])
        r[11:11 + len(nd["out_axes"])] = nd["out_axes"]
        w = nd.get("w_axes") or []
        r[19] = len(w)
        r[20:20 + len(w)] = w
        fd = nd.get("flop_dims")
        r[28] = 0 if fd is None else sum(1 << k for k in fd)
        r[29] = nd.get("flops_per_point", 2)
        halo = nd.get("halo") or []
        r[30] = len(halo)
        for q, (h, f) in enumerate(halo):
            r[31 + q], r[35 + q] = h, f
        r[39] = nd.get("elem_bytes", 4)
        ins = nd.get("in_axes") or []
        r[40] = len(ins)
        r[41:41 + len(ins)] = ins
    edges = graph["edges"]
    E = np.full((max(len(edges), 1), EDGE_REC), -1, dtype=np.int64)
    for e, ed in enumerate(edges):
        E[e, 0], E[e, 1] = ed["src"], ed["dst"]
        am = ed["axis_map"]
        E[e, 2:2 + len(am)] = am
    return N, E


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def _chk(rc: int, what: str) -> None:
    if rc != 0:
        raise OracleError(rc, what)


def validate(graph: dict) -> int:
    N, E = encode(graph)
    return lib().or_validate(len(N), _p(N, C.c_int64), len(graph["edges"]), _p(E, C.c_int64))


def configs(graph: dict, p: int, policy: int = EXACT_P) -> List[np.ndarray]:
    N, _ = encode(graph)
    n = len(N)
    K = np.zeros(n, dtype=np.int32)
    _chk(lib().or_configs(n, _p(N, C.c_int64), p, policy, _p(K, C.c_int32), None), "configs")
    T = np.zeros((int(K.sum()), MAXD), dtype=np.int32)
    _chk(lib().or_configs(n, _p(N, C.c_int64), p, policy, _p(K, C.c_int32), _p(T, C.c_int32)), "configs")
    out, off = [], 0
    for v in range(n):
        d = len(graph["nodes"][v]["dims"])
        out.append(T[off:off + K[v], :d].copy())
        off += K[v]
    return out


def cost_tables(graph: dict, p: int, policy: int = EXACT_P,
                machine: Optional[dict] = None) -> Tuple[np.ndarray, List[np.ndarray], List[np.ndarray]]:
    """Returns (K, [L_v], [W_e as K_src x K_dst])."""
    machine = machine or graph.get("machine") or {"flops": 1e13, "bandwidth": 1e10}
    N, E = encode(graph)
    n, m = len(N), len(graph["edges"])
    K = np.array([len(c) for c in configs(graph, p, policy)], dtype=np.int32)
    L = np.zeros(int(K.sum()), dtype=np.float64)
    wsz = sum(int(K[e["src"]]) * int(K[e["dst"]]) for e in graph["edges"])
    W = np.zeros(max(wsz, 1), dtype=np.float64)
    _chk(lib().or_cost_tables(n, _p(N, C.c_int64), m, _p(E, C.c_int64), p, policy,
                              float(machine["flops"]), float(machine["bandwidth"]),
                              _p(L, C.c_double), _p(W, C.c_double)), "cost_tables")
    Ls, off = [], 0
    for v in range(n):
        Ls.append(L[off:off + K[v]].copy())
        off += K[v]
    Ws, off = [], 0
    for e in graph["edges"]:
        ks, kt = int(K[e["src"]]), int(K[e["dst"]])
        Ws.append(W[off:off + ks * kt].reshape(ks, kt).copy())
        off += ks * kt
    return K, Ls, Ws


class Problem:
    """Graph topology + explicit cost tables (memoised t_l / r*t_x, or synthetic)."""

    def __init__(self, graph: dict, K, Ls, Ws):
        self.graph = graph
        _, self.E = encode(graph)
        self.n, self.m = len(graph["nodes"]), len(graph["edges"])
        self.K = np.ascontiguousarray(K, dtype=np.int32)
        self.L = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64).ravel() for x in Ls]))
        ws = [np.asarray(x, np.float64).ravel() for x in Ws]
        self.W = np.ascontiguousarray(np.concatenate(ws) if ws else np.zeros(1))
        self.Ls, self.Ws = [np.asarray(x, np.float64) for x in Ls], [np.asarray(x, np.float64) for x in Ws]

    @classmethod
    def from_model(cls, graph: dict, p: int, policy: int = EXACT_P, machine: Optional[dict] = None):
        K, Ls, Ws = cost_tables(graph, p, policy, machine)
        return cls(graph, K, Ls, Ws)

    def _args(self):
        return (self.n, self.m, _p(self.E, C.c_int64), _p(self.K, C.c_int32),
                _p(self.L, C.c_double), _p(self.W, C.c_double))

    def sortnodes(self) -> Tuple[np.ndarray, List[List[int]]]:
        sigma = np.zeros(self.n, np.int32)
        off = np.zeros(self.n + 1, np.int32)
        ids = np.zeros(self.n * self.n + 1, np.int32)
        _chk(lib().or_sortnodes(self.n, self.m, _p(self.E, C.c_int64), _p(sigma, C.c_int32),
                                _p(off, C.c_int32), _p(ids, C.c_int32)), "sortnodes")
        return sigma, [list(ids[off[i]:off[i + 1]]) for i in range(self.n)]

    def bfs_order(self) -> np.ndarray:
        sigma = np.zeros(self.n, np.int32)
        _chk(lib().or_bfs_order(self.n, self.m, _p(self.E, C.c_int64), _p(sigma, C.c_int32)), "bfs")
        return sigma

    def sets(self, sigma, i: int) -> Dict[str, object]:
        n = self.n
        sigma = np.ascontiguousarray(sigma, np.int32)
        X, D, Db = (np.zeros(n, np.uint8) for _ in range(3))
        comp = np.zeros(n, np.int32)
        nc = np.zeros(1, np.int32)
        _chk(lib().or_sets(n, self.m, _p(self.E, C.c_int64), _p(sigma, C.c_int32), i,
                           _p(X, C.c_uint8), _p(D, C.c_uint8), _p(Db, C.c_uint8),
                           _p(comp, C.c_int32), _p(nc, C.c_int32)), "sets")
        S = [set(np.nonzero(comp == c)[0].tolist()) for c in range(int(nc[0]))]
        return {"X": set(np.nonzero(X)[0].tolist()), "D": set(np.nonzero(D)[0].tolist()),
                "Dbar": set(np.nonzero(Db)[0].tolist()), "S": S}

    def table_sizes(self, order: int = 0) -> Tuple[np.ndarray, int]:
        off = np.zeros(self.n + 1, np.int64)
        cand = np.zeros(1, np.int64)
        _chk(lib().or_table_sizes(self.n, self.m, _p(self.E, C.c_int64), _p(self.K, C.c_int32), order,
                                  _p(off, C.c_int64), _p(cand, C.c_int64)), "table_sizes")
        return off, int(cand[0])

    def dp(self, order: int = 0, threads: int = 1, table_limit: int = 0, want_tables: bool = False):
        """Fig. 5 DP-Alg.  Returns dict(strategy, cost, seconds[, T, A, toff])."""
        strat = np.zeros(self.n, np.int32)
        tot = np.zeros(1, np.float64)
        T = A = None
        off = None
        if want_tables:
            off, _ = self.table_sizes(order)
            T = np.zeros(int(off[-1]), np.float64)
            A = np.zeros(int(off[-1]), np.int32)
        t0 = time.perf_counter()
        rc = lib().or_dp(*self._args(), order, threads, table_limit, _p(strat, C.c_int32), _p(tot, C.c_double),
                         _p(T, C.c_double) if T is not None else None,
                         _p(A, C.c_int32) if A is not None else None)
        dt = time.perf_counter() - t0
        _chk(rc, "dp")
        out = {"strategy": strat, "cost": float(tot[0]), "seconds": dt}
        if want_tables:
            out.update(T=T, A=A, toff=off)
        return out

    def dp_select(self, ranks, threads: int = 1, order: int = 0):
        """Fig. 5 DP-Alg returning only the tables of `ranks`: dict(strategy, cost, seconds,
        tables={rank: (T, A)})."""
        off, _ = self.table_sizes(order)
        ranks = [int(r) for r in ranks]
        sizes = [int(off[r + 1] - off[r]) for r in ranks]
        T = np.zeros(max(sum(sizes), 1), np.float64)
        A = np.zeros(max(sum(sizes), 1), np.int32)
        sel = np.ascontiguousarray(ranks, np.int32)
        strat = np.zeros(self.n, np.int32)
        tot = np.zeros(1, np.float64)
        t0 = time.perf_counter()
        rc = lib().or_dp_select(*self._args(), order, threads, _p(strat, C.c_int32), _p(tot, C.c_double),
                                len(ranks), _p(sel, C.c_int32), _p(T, C.c_double), _p(A, C.c_int32))
        dt = time.perf_counter() - t0
        _chk(rc, "dp_select")
        tables, o = {}, 0
        for r, sz in zip(ranks, sizes):
            tables[r] = (T[o:o + sz], A[o:o + sz])
            o += sz
        return {"strategy": strat, "cost": float(tot[0]), "seconds": dt, "tables": tables}

    def dp_bfs_eq2(self, table_limit: int = 0):
        strat = np.zeros(self.n, np.int32)
        tot = np.zeros(1, np.float64)
        _chk(lib().or_dp_bfs_eq2(*self._args(), table_limit, _p(strat, C.c_int32), _p(tot, C.c_double)), "dp_bfs_eq2")
        return {"strategy": strat, "cost": float(tot[0])}

    def brute(self, limit: int = 10 ** 8):
        strat = np.zeros(self.n, np.int32)
        tot = np.zeros(1, np.float64)
        _chk(lib().or_brute(*self._args(), limit, _p(strat, C.c_int32), _p(tot, C.c_double)), "brute")
        return {"strategy": strat, "cost": float(tot[0])}

    def eval(self, strategy) -> float:
        s = np.ascontiguousarray(strategy, np.int32)
        return lib().or_eval(*self._args(), _p(s, C.c_int32))

    def sum_h(self, sigma, strategy) -> float:
        s = np.ascontiguousarray(strategy, np.int32)
        sg = np.ascontiguousarray(sigma, np.int32)
        return lib().or_sum_h(*self._args(), _p(sg, C.c_int32), _p(s, C.c_int32))


def assign_devices(graph: dict, p: int, tuples) -> Tuple[np.ndarray, np.ndarray]:
    """f3: greedy device assignment of a strategy given as config tuples per node
    (P:288-294).  Returns (dev int32[n, p] with -1 padding, realized t_x bytes float64[m])."""
    N, E = encode(graph)
    n, m = len(N), len(graph["edges"])
    cfg = np.ones((n, MAXD), np.int32)
    for v, t in enumerate(tuples):
        cfg[v, :len(t)] = t
    dev = np.zeros((n, p), np.int32)
    tx = np.zeros(max(m, 1), np.float64)
    _chk(lib().or_assign(n, _p(N, C.c_int64), m, _p(E, C.c_int64), p, _p(cfg, C.c_int32), _p(dev, C.c_int32),
                         _p(tx, C.c_double)), "or_assign")
    return dev, tx[:m]
