"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain numpy (f32/f64) restatement of the reference's scoring path, used as the parity checker
for the B200 kernels.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it; the product package
(``paper_2510_22101_b200``) never does.

What it restates (all citations into /root/reference):
  model.py       SPEC.md:172-238  ModelConfig / Weights / init_weights / forward_prefill /
                                  forward_with_prefix / KVCache
  prefixcache.py SPEC.md:240-309  split_shared_prefix / merge_attention / score_shared_batch /
                                  throughput_gain, plus the flat packer layout the device uses
  scoring.py     SPEC.md:311-343  relevance_score (Eq 2) / rank_items
  calibration.py SPEC.md:458-485  capture_calibration sampling, direct least-squares greedy backward
                                  elimination and the exhaustive optimum (OSSCAR stand-in checks)
  tokenizer.py   pkg/src/prefrank/tokenizer.py  encode / encode_with_spans / word_id, restated as an
                                  explicit scanner; pinned to the reference-generated goldens
  The reference package ships NO code for these modules: the model path is
  "parity unpinned" by reference-executed outputs.  It is pinned by the spec's known-answer
  examples and invariants (tests/test_oracle.py) and the token-id / prompt-structure golden
  vectors generated from the importable reference tokenizer.py + corpus.py
  (tests/golden/make_golden.py).  Its transformer arithmetic is additionally pinned against an
  independent implementation: Hugging Face transformers' LlamaForCausalLM in float64 on the same
  weights agrees to ~1e-14 on last-token logits (tests/golden/make_hf_llama_golden.py ->
  hf_llama_logits.json; tests/test_oracle_hf.py), for the C1 shape, a GQA model with
  n_heads*d_head != d_model and a 10/5-head pruned shape, including the prefix-shared path.

Open choices the spec leaves (pinned identically in the product): pre-norm blocks,
RMSNorm eps 1e-6, rotate-half RoPE with theta^(-2i/d_head) tables computed in float64, GQA head
h -> kv head h // (H/Hkv), scale 1/sqrt(d_head), PCG64 init with the draw order in model.py,
unit norm scales, bf16-representable weight values.
"""
