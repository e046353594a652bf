"""ORACLE — plain, slow, obviously-correct CPU fp64 implementation of the MRAB / SBP-SAT
overset hot path of arXiv 1805.06607 (Mikida, Kloeckner, Bodony).

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The product path
(`paper_1805_06607_b200`, `libmrab.so`) never imports, links or calls anything in here, and
this package never imports the product.  The two share no code; only the seeded input
generators in `synth/` (which hold none of the method's arithmetic) serve both.

Every function cites the PAPER.md passage (P:<line>) it follows, or the numbered reading
of DESIGN.md §2 (R<k>, which restate SURVEY.md §8(c)'s G-readings) where the paper is
silent or garbled.

Modules
  sbp       SBP 2-4 diagonal-norm D1, segments, norm H
  abcoef    AB / extended-history AB weights in exact rationals
  gas       primitives, inviscid / viscous fluxes, K^+- matrices
  metrics   conservative curvilinear metric terms                (reading R3)
  overset   hole cutting, donor search, Lagrange weights         (reading R17)
  rhs       the coupled SBP-SAT right-hand side of all meshes    (eq:int P:279-299)
  timeint   RK3/RK4 bootstrap, N-rate fastest-first MRAB

Parity pins: see tests/test_oracle_*.py and DESIGN.md §4.  Functions without an
independent pin say "parity unpinned" in their docstring.
"""
