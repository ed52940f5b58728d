"""Golden fixture for the profiler objective, from the
reference's OWN profiler.cpp / proxy.cpp compiled in place (oracle/_ref; needs
/root/reference in this container):

  objective.npz   simulated ProxyBatch features (proxy.cpp simulate, three
                  regimes), the reference's build_proxy_cache row sums and
                  |A_dense|_F^2, and objective() = (loss, mse, sparsity) for
                  static and dynamic configurations.

    python tests/golden/make_objective_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle  # noqa: E402
from oracle.pyoracle import Cfg  # noqa: E402

NF, NT, BS, DIM = 6, 96, 16, 32
SEEDS = (11, 12, 13)
# (mode, gamma, lambda, split_eps, theta_m, theta_c, near, far, fallback_k)
CONFIGS = [
    (0, 1.5, 0.5, 1e-6, 0.6, 0.3, 0.5, 0.3, 1),
    (0, 2.0, 1.0, 1e-6, 0.9, 0.9, 0.1, 0.1, 1),
    (0, 1.0, 1.0, 1e-6, 0.2, 0.1, 1.0, 0.8, 1),
    (1, 1.5, 0.5, 1e-6, 0.6, 0.3, 0.0, 1.0, 1),
    (1, 2.5, 0.2, 1e-6, 0.3, 0.2, -1.0, 0.5, 2),
    (1, 1.2, 0.9, 1e-6, 0.3, 0.2, 0.5, 1.0, 1),
]


def main():
    R = pyoracle.ref()
    feats, rows, sqs, outs = [], [], [], []
    for regime, seed in enumerate(SEEDS):
        f = R.simulate(NF, NT, BS, DIM, seed, regime=regime)
        _, rs, sq = R.proxy_cache(NF, NT, BS, f)
        feats.append(f)
        rows.append(rs)
        sqs.append(sq)
        outs.append([R.objective(NF, NT, BS, Cfg(*c), f, seed, 10.0, 0.8) for c in CONFIGS])
    np.savez_compressed(os.path.join(HERE, "objective.npz"), nf=NF, nt=NT, bs=BS, dim=DIM,
                        seeds=np.array(SEEDS, np.uint64), features=np.stack(feats),
                        row_sums=np.stack(rows), sq_norm=np.array(sqs),
                        configs=np.array(CONFIGS, np.float64), trials=np.array(outs))
    print("objective.npz:", np.array(outs)[:, :, 1])


if __name__ == "__main__":
    main()
