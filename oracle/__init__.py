"""FlashSampling CPU oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation of what the fused
LM-head + exact Gumbel-max sampling path computes (arXiv 2603.15854, PAPER.md).

Rules:
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
    leg may import this package.  The product package (paper_2603_15854_b200) never
    imports it and has no CPU fallback.
  * It shares no code with the CUDA path: its own Philox4x32-10, its own Gumbel
    evaluation, its own transform and argmax.  Only `synth` (seeded inputs, no
    method arithmetic) is common to both sides.
  * Every function cites the PAPER.md passage it follows ("P:<line>").

Modules
  philox     Philox4x32-10 counter-based generator (P:195-197 names "e.g. Philox").
  rng        counter layout (reading R1) and the exact-math Gumbel map (App. C).
  sampler    flat fused-path definition (Alg. 2, as argmax over the whole row,
             Lemma P:365-391), grouped summaries (§4.1, Lemma P:254-289), TP
             shards (Alg. A.4) and log-normalizer (App. E).
  variants   the in-distribution algorithms (Alg. 1, A.1 P:747-763, A.2 P:768-784,
             A.3 P:789-815, A.4 P:820-836 with fresh outer Gumbels / Bernoulli merge).
  stats      chi-square goodness of fit (§5.7) and Gumbel moment checks.
  costmodel  §4.7 cost model.

Parity status (pins in tests/test_oracle_*.py):
  philox, rng.gumbel64, sampler.*, variants.*, costmodel.*: pinned.
  The specific sampled index for given (seed, step) is "parity unpinned" against the
  paper (the paper prints no RNG stream or sampled index); it is pinned against the
  exact definition via an independent Decimal evaluation of the Gumbel map on tiny
  hand-checkable inputs (tests/golden/).
"""
