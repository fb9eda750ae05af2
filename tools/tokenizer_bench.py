"""Tokenizer throughput: native C++ (libprefill_sm100.so) vs the reference Python encode_batch.
Needs /root/reference (build container only).   python tools/tokenizer_bench.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
from prefrank import corpus, tokenizer
from paper_2510_22101_b200 import ingest

qs, items = corpus.generate_corpus(7, 20, 500)
vocab = tokenizer.Vocab()
texts = [corpus.assemble_prompt(qs[i % 20], it).full_prompt() for i, it in enumerate(items)] * 4
t0 = time.perf_counter(); ref = tokenizer.encode_batch(texts, vocab); t_ref = time.perf_counter() - t0
ntok = sum(len(x) for x in ref)
for nt in (1, os.cpu_count()):
    t0 = time.perf_counter(); ids, offs = ingest.encode_batch_arrays(texts, n_threads=nt); t = time.perf_counter() - t0
    assert len(ids) == ntok
    print(f"native threads={nt}: {ntok / t / 1e6:.1f} M tok/s")
print(f"reference encode_batch (Python): {ntok / t_ref / 1e6:.2f} M tok/s  ({len(texts)} prompts, {ntok} tokens)")
