"""Subprocess body of tests/test_gpu_variants.py: bit-exact parity (every cost table, every
DP table, strategy, total) of the CUDA path against the oracle under the PASE_* switches in
the environment (they are read once per process)."""
import sys

import numpy as np

from oracle import oracle as O
from paper_2407_04001_b200 import zoo
from tests.helpers import random_costs
from tests.test_gpu_parity import run_pair


def main():
    for name in sys.argv[1].split(","):
        g, p = zoo.bench_graph(name)
        run_pair(g, p, "exact_p")
    for seed in range(int(sys.argv[2])):
        g = zoo.random_model_graph(2 + seed % 9, 900 + seed, multi_p=0.15 if seed % 4 == 0 else 0.0)
        run_pair(g, 4 << (seed % 3), "exact_p" if seed % 2 else "le_p")
        g, p = zoo.random_chain_graph(1 + seed % 8, 1900 + seed, kmax=12, extra_p=0.4)
        K = np.array([len(c) for c in O.configs(g, p, O.LE_P)], np.int32)
        Ls, Ws = random_costs(g, K, 3000 + seed, "int" if seed % 2 else "real")
        run_pair(g, p, "le_p", Ls, Ws)
    print("variant parity ok")


if __name__ == "__main__":
    main()
