"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Holds none of the method's arithmetic: only random vectors and size recipes
(SURVEY.md §8d "Inputs").  x, b ~ U[-1, 1) i.i.d. in FP64 from
numpy PCG64 with seed_x = 20241205, seed_b = 20241206; FP32 runs use RN-rounded copies.
"""
import numpy as np

SEED_X = 20241205
SEED_B = 20241206


def n_dofs(k, d, N):
    """Interior DoFs (k N - 1)^d of level N (clamped boundary nodes eliminated)."""
    return (k * N - 1) ** d


def uniform(n, seed):
    """n i.i.d. U[-1, 1) FP64 values from PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=n)


def random_xb(k, d, N, seed_x=SEED_X, seed_b=SEED_B):
    n = n_dofs(k, d, N)
    return uniform(n, seed_x), uniform(n, seed_b)


def sample_ids(n, count, seed=7):
    """Sorted distinct sample indices for sampled parity at full sizes."""
    rng = np.random.Generator(np.random.PCG64(seed))
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False))


# Throughput meshes of SURVEY.md §8d (cfg2: ~16.7M DoFs 2D; cfg4: ~50M DoFs 3D)
CFG2_CELLS = {2: 2048, 3: 1365, 4: 1024, 5: 819, 6: 683, 7: 585}
CFG4_CELLS = {2: 184, 3: 123, 4: 92, 5: 74}
