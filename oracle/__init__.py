"""nuGPR oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, FP64 CPU implementation of what the nuGPR training hot path computes
(arXiv 2510.12128, /root/reference/PAPER.md), written from the paper in its order and
notation.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product path (`paper_2510_12128_b200/`)
never imports, links or executes anything here, and this package shares no code with
it (the only common module is `synth/`, which draws inputs and holds none of the
method's arithmetic).

Modules
  kernels     Eq. (2) RBF (squared-distance reading X3/P1), the as-printed form, Matern-5/2
  structured  Eq. (12)-(13) block Cholesky + jitter, Eq. (21) u_i, Eq. (26)-(28) K_rep,
              lambda_0, M; the preconditioned operator A with the Eq. (23)-(25) shortcuts
  cg          §3.1 CG / batched CG with per-column freezing (readings P3-P7)
  logdet      Eq. (9)-(10), (16) Hutchinson + Pade trace; SLQ from the CG coefficients
  mll         Eq. (3) loss assembly; Eq. (11) numerical gradient (CENTRAL, FORWARD_HALVING);
              Adam; Algorithm 1 training loop
  exact       O-EXACT (Woodbury + determinant lemma) and O-DENSE (dense Cholesky) exact
              structured MLL, analytic gradient — the oracle's own cross-checks
  kmeans      A0: Lloyd k-means with fixed-point centroid sums (reading P18)
  predict     Eq. (4)-(7) posterior mean / variance (NEXT-1)

Parity pins (tests/test_oracle_*.py) tie every function to something other than
itself; see DESIGN.md "Oracle pins".  Parity unpinned (pinned only by running the
same algorithm on the same inputs): the tol-stopped iteration counts, the Hutchinson
realisation, the FORWARD_HALVING stopping decisions and the Adam trajectory.
"""
