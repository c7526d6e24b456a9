"""DoF numbering, vertex patches and colours (Fig. 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings: C1 numbering (interior nodes only, x fastest), C2 patch
numbering (vertex v in [1,N-1]^d, patch id sum_a (v_a-1)(N-1)^a), C3 colours
(colour = 2 * parity-class + red-black key, parity class = sum_a (v_a mod 2) 2^a,
red-black key = (sum_a floor(v_a/2)) mod 2; readings Q14, Q15).  Levels: N = 2^level
(reading Q9).
"""
import itertools
import numpy as np


def level_cells(level):
    """Reading Q9: level l has N = 2^l cells per axis; level 1 is the 2^d-cell mesh."""
    return 2 ** level


def n_dofs_1d(k, N):
    return k * N - 1


def patch_vertices(d, N):
    """[(N-1)^d, d] vertex multi-indices in patch-id order (v_x fastest)."""
    return np.array(list(itertools.product(range(1, N), repeat=d)))[:, ::-1]


def patch_dofs(k, d, N, v):
    """Global interior DoF ids of patch v (patch-local order, x fastest): R_v."""
    n = n_dofs_1d(k, N)
    ranges = [np.arange((va - 1) * k, (va + 1) * k - 1) for va in v]
    idx = np.zeros([2 * k - 1] * d, dtype=np.int64)
    for a in range(d):
        shape = [1] * d; shape[d - 1 - a] = 2 * k - 1
        idx = idx + (ranges[a] * n ** a).reshape(shape)
    return idx.ravel()


def all_patch_dofs(k, d, N):
    """[(N-1)^d, (2k-1)^d] DoF map of every patch."""
    return np.array([patch_dofs(k, d, N, v) for v in patch_vertices(d, N)], dtype=np.int64)


def color_of(v):
    """Reading Q14/Q15 colour of vertex v: 2 * sum_a (v_a mod 2) 2^a + (sum_a floor(v_a/2)) mod 2."""
    v = np.asarray(v)
    parity = sum(int(v[a] % 2) << a for a in range(len(v)))
    rb = int(sum(int(va) // 2 for va in v) % 2)
    return 2 * parity + rb


def n_colors(d):
    """8 colours in 2D, 16 in 3D."""
    return 2 ** (d + 1)


def color_patches(d, N):
    """List over colours (ascending) of patch ids in that colour, lexicographic."""
    verts = patch_vertices(d, N)
    cols = np.array([color_of(v) for v in verts])
    return [np.nonzero(cols == c)[0] for c in range(n_colors(d))]
