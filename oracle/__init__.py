"""ORACLE — test infrastructure, NOT part of the product path.

A plain, slow, serial float64 CPU implementation of what the AIFMM hot path
computes, written from the paper (/root/reference/PAPER.md, cited as P:<line>
with its section / equation / algorithm).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
leg may import it.  It shares no code with the CUDA path
(`paper_2301_12704_b200/`); the only common module is the seeded input
generator `paper_2301_12704_b200/workloads.py`, which holds none of the
method's arithmetic.

Modules
  tree     §2.1 tree, Morton numbering, N(i)/IL(i), colouring
  kernels  matrix entries A_ij = K(x_i, x_j)
  linalg   tie-window argmax, pivoted Gram-Schmidt QR with truncation (RRQR)
  nnca     NNCA pivots and operators (Eq. NCA, operators P:360-367)
  factor   extended sparse system (§3.1), colour-batched Algorithm 3
           with compression/redirection (§3.2.1-3.2.3), top solve, Algorithm 4
  dense    dense references (direct LU solve, densified NNCA/H2 matrix, residuals)

Every reading of the paper that is not literal is listed in DESIGN.md
("Readings") and referenced here as R<n>.
"""
