"""Seeded synthetic cost tables and graph utilities shared by the tests.

Holds none of the method's arithmetic (no ordering, no DP, no cost model): only
random numbers and graph relabelling.  Random numbers the method consumes are
drawn here and passed to BOTH sides as inputs.
"""
from __future__ import annotations

import copy
import random
from typing import List, Tuple

import numpy as np


def random_costs(graph: dict, K, seed: int, kind: str = "int") -> Tuple[List[np.ndarray], List[np.ndarray]]:
    """L_v[K_v] and W_e[K_src, K_dst].  kind='int': integers 0..1000 stored as fp64
    (exact sums, exercises ties); kind='real': U[0,1) (exercises summation order)."""
    rng = np.random.default_rng(seed)
    Ls, Ws = [], []
    for v in range(len(graph["nodes"])):
        if kind == "int":
            Ls.append(rng.integers(0, 1001, int(K[v])).astype(np.float64))
        else:
            Ls.append(rng.random(int(K[v])))
    for e in graph["edges"]:
        shape = (int(K[e["src"]]), int(K[e["dst"]]))
        if kind == "int":
            Ws.append(rng.integers(0, 1001, shape).astype(np.float64))
        else:
            Ws.append(rng.random(shape))
    return Ls, Ws


def relabel(graph: dict, seed: int) -> Tuple[dict, List[int]]:
    """Permute node ids (new id = perm[old id]); edges keep their order."""
    n = len(graph["nodes"])
    perm = list(range(n))
    random.Random(seed).shuffle(perm)
    g2 = copy.deepcopy(graph)
    nodes = [None] * n
    for old, nd in enumerate(graph["nodes"]):
        nn = copy.deepcopy(nd)
        nn["id"] = perm[old]
        nodes[perm[old]] = nn
    g2["nodes"] = nodes
    for e in g2["edges"]:
        e["src"], e["dst"] = perm[e["src"]], perm[e["dst"]]
    return g2, perm


def degrees(graph: dict) -> List[int]:
    n = len(graph["nodes"])
    nb = [set() for _ in range(n)]
    for e in graph["edges"]:
        nb[e["src"]].add(e["dst"])
        nb[e["dst"]].add(e["src"])
    return [len(x) for x in nb]
