"""Seeded synthetic requests (SURVEY.md §8d "Synthetic inputs").

Prefix ids start with 3 (<|sys|>) and are uniform in the hashed-word range [16, 32768)
(tokenizer.py:76); suffix ids likewise.  Family "template": every suffix ends in 11 (<|ans|>,
Eq 1, corpus.py:31).  Family "spread": random last token (strict top-k parity family).
"""

import numpy as np

ANS_ID = 11
SYS_ID = 3


def make_prompts(rng, prefix_len, suffix_lens, family="template", vocab=32768):
    prefix = [SYS_ID] + list(rng.integers(16, vocab, prefix_len - 1)) if prefix_len > 0 else []
    prompts = []
    for s in suffix_lens:
        suf = list(rng.integers(16, vocab, s))
        if family == "template":
            suf[-1] = ANS_ID
        prompts.append([int(t) for t in prefix] + [int(t) for t in suf])
    return prompts


def make_shared(rng, prefix_len, suffix_lens, family="template", vocab=32768):
    from paper_2510_22101_b200.prefixcache import split_shared_prefix

    sb = split_shared_prefix(make_prompts(rng, prefix_len, suffix_lens, family, vocab))
    return sb
