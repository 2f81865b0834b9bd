"""CPU oracle for CAKF/CAKS (arXiv 2405.08971) — TEST INFRASTRUCTURE ONLY.

Plain, slow, dense fp64 numpy/scipy implementations of what the hot path
computes, written from PAPER.md (cited per function as "P:<line>").  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything in this package.  The
product path (``paper_2405_08971_b200``) never imports it and shares no code,
constants or helpers with it; both consume inputs from ``synth/`` only.

Modules
  model   — Matérn SDE (expm + Lyapunov), spatial kernels, dense Kronecker LGSSM
  kf      — exact Kalman filter, RTS smoother, downdate-form KF, inverse-free RTS,
            brute-force joint-Gaussian conditioning
  cakf    — dense CAKF (alg:mfkf + alg:update_pls + Truncate), batch update
            (alg:projected_update), dense CAKS (alg:mfks)
  itergp  — exact and iteratively-approximated batch GP posterior (Def. B.3)
  philox  — Philox4x32-10 counter-based generator for random actions (R16)
  mfree   — matrix-free chunked CAKF/CAKS (same algorithm, kernel rows generated
            per chunk) for state dimensions where dense matrices do not fit

Parity status of every function is listed in DESIGN.md §4 ("pinned by").
"""
