"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (numpy float64) implementation of the
server-side verify step of arXiv 2505.21594 ("speculative edge-cloud decoding
with early exits"): one Llama-style decoder pass over gamma+1 query tokens
against a KV cache (Eq. 3 and LMHead), an early-exit head at an
intermediate layer (Eq. 5; Eq. 4 confidence PAPER.md:104-107),
Leviathan speculative-sampling acceptance (Eq. 2, adopted by
citation PAPER.md:24, :80) and KV rollback to the accepted length.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything in this package.  The
product path (`paper_2505_21594_b200`) never imports it and shares no code with
it; the only shared module is `workload/` (seeded input generators, no method
arithmetic).

Modules
  philox   Philox4x32-10 counter-based generator (Salmon et al. 2011) + uniforms
  gen      counter-hash weight / synthetic-KV generator (bf16, bit-defined)
  model    fp64 Llama forward with a KV cache, exit head and final head
  accept   greedy / stochastic acceptance, residual, confidence, exit score
  verify   one verify step for a session: forward + exit + accept + rollback

Parity pins live in tests/test_oracle_*.py.  Functions without a pin say
"parity unpinned" in their docstring.
"""
