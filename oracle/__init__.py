"""CPU oracle for hidden-state tree speculative decoding (arXiv 2602.21224).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this package.
The product path (`paper_2602_21224_b200`) never imports it and shares no code
with it: the two sides agree only through the published Philox4x32-10 generator
(implemented independently on each side) and the inputs produced by `synth`.

Plain, slow, obviously-correct numpy in float64. Each function cites the
PAPER.md passage it follows (P:<line>, section / equation / algorithm), or the
DESIGN.md reading (R<k>) where the paper is silent.

Pins (tests/test_oracle_*.py):
  philox   - Random123 published known-answer vectors.
  model    - HuggingFace `transformers` LlamaForCausalLM in float64 on the same
             weights (an independent Llama implementation).
  attention- torch scaled_dot_product_attention (float64) per root path.
  table    - PAPER.md:168 "15.3 GB" at |V|=128,256 FP8; "1/16";
             row RMS = 1; cold rows/cols exactly 0; W_E[t]·W1·W2 by brute force.
  fp8      - e4m3 table rows (R25): the 254 finite codes decoded bit by bit,
             torch float8_e4m3fn cast, ties to even, saturation, row amax = 448.
  tree     - Fig. 5 worked example: 0.6, 0.3, 0.42, 0.294;
             k=1 greedy chain; zero table == beam tree; independent recursive
             brute-force builder; node-count bound.
  prune    - sort-all-nodes brute force + connectivity.
  resample - Alg. 2 reduces to Alg. 1 on the truncated chain / single node.
  fuse     - path-set union.
  engine   - greedy losslessness: speculative output == plain greedy decode.
  accept   - stochastic: chi-square of emitted tokens vs softmax(target logits).
  compaction - committed KV == the KV a plain decode writes.
"""
