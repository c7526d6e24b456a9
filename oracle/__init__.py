"""CPU oracle for the C0IP vertex-patch Schwarz smoother (arXiv 2412.05082).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2412_05082_b200``) never imports it, and this
package never imports the product path: the two share no code.  The only shared
module is ``c0ip_inputs`` (seeded random inputs, no method arithmetic).

The oracle is plain and slow on purpose: FP64 NumPy/SciPy, an *assembled* sparse
C0IP matrix built by d-dimensional cell and face quadrature (never the Kronecker
identity), dense per-patch surrogate matrices solved by Cholesky (never fast
diagonalisation), and textbook V-cycle / CG loops.  Every function cites the
PAPER.md line (section / equation / algorithm) it follows; ambiguous readings are
the ones listed in SURVEY.md §8(c) (Q1-Q26) and DESIGN.md.

Modules
-------
basis         Gauss-Lobatto Lagrange basis and Gauss quadrature on [0,1]
discretization 1D matrices M, L, B (Eq. matrix1d) by 1D quadrature
operator      d-dim C0IP assembly (Eq. bfc0ip), window rows, loads
mesh          DoF numbering, vertex patches, colours
smoothers     dense surrogate patch solves, AVS / MVS steps
multigrid     transfers, V-cycle (Alg. 1), PCG and nu
"""
