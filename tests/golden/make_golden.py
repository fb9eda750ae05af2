"""Generate tests/golden/prompts.json from the REFERENCE package (run in the build container only;
/root/reference does not exist on the GPU box — the committed JSON travels instead).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference's own tokenizer.py and corpus.py (the only executable parts of the path,
SURVEY.md §0) and records:
  * the Vocab special-id table and FNV-1a constants (tokenizer.py:22-37, :49-76);
  * encode() known answers (SYSTEM_PREFIX, "<|ans|>", "yes", "no", "rust engineer", "");
  * Eq-1 prompts (corpus.assemble_prompt, corpus.py:302-311) for seeded queries x items, truncated
    to the 2048-token budget (corpus.truncate_description, corpus.py:314-345), as token ids, plus the
    per-segment token counts — the golden inputs for split_shared_prefix / packing parity;
  * a truncation known answer (budget 300) and the PromptBudgetError message for a tiny budget.
"""

import json
import os
import sys

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import random  # noqa: E402

from prefrank import corpus, tokenizer  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "prompts.json")


def main():
    vocab = tokenizer.Vocab()
    enc = lambda s: tokenizer.encode(s, vocab)
    queries, items = corpus.generate_corpus(7, 4, 40)
    requests = []
    for qi, q in enumerate(queries):
        cands = items[qi * 8: qi * 8 + 8]
        prompts, seg_lens = [], []
        for it in cands:
            seg = corpus.truncate_description(corpus.assemble_prompt(q, it), 2048, vocab)
            full = enc(seg.full_prompt())
            parts = [enc(seg.system_prefix), enc(seg.query_text), enc(seg.metadata_text),
                     enc(seg.description_text), enc(seg.suffix)]
            assert sum(parts, []) == full
            prompts.append(full)
            seg_lens.append([len(p) for p in parts])
        requests.append({"query_id": q.id, "item_ids": [it.id for it in cands],
                         "prompts": prompts, "segment_lens": seg_lens})
    seg = corpus.assemble_prompt(queries[0], items[0])
    trunc300 = enc(corpus.truncate_description(seg, 300, vocab).full_prompt())
    try:
        corpus.truncate_description(seg, 10, vocab)
        budget_err = None
    except corpus.PromptBudgetError as e:
        budget_err = str(e)
    # tokenizer known answers on adversarial texts: case, punctuation, tag spellings, Unicode whose
    # lowercase is ASCII (U+0130, U+212A), other scripts, combining marks, emoji
    frng = random.Random(2510)
    alphabet = (list("abcxyzABCXYZ0189 _-.,;:!?|<>/\\'\"()[]{}\t\n") + ["<|sys|>", "<|/SYS|>", "<|Q|>", "<|/q|>",
                "<|meta|>", "<|/meta|>", "<|desc|>", "<|/desc|>", "<|ANS|>", "<|ans", "|>", "<|",
                "\u0130", "\u212a", "\u00df", "\u00c9", "\u0131", "\u03a3", "\u4e2d\u6587", "\u0307",
                "\U0001F600", "yes", "no", "Yes", "NO", "rust", "Engineer"])
    fuzz = ["".join(frng.choice(alphabet) for _ in range(frng.randint(0, 60))) for _ in range(400)]
    fuzz += ["", "   ", "\u0130stanbul KELVIN \u212a", "<|ans|><|ans|>", "a<|q|>b", "x" * 300]
    prompt_texts = []
    for qi, q in enumerate(queries[:2]):
        for it in items[qi * 8: qi * 8 + 3]:
            prompt_texts.append(corpus.truncate_description(corpus.assemble_prompt(q, it), 2048, vocab).full_prompt())
    from dataclasses import asdict
    assembly = []
    for qi, q in enumerate(queries[:2]):
        for it in items[qi * 8: qi * 8 + 4]:
            seg = corpus.assemble_prompt(q, it)
            base = sum(len(enc(x)) for x in (seg.system_prefix, seg.query_text, seg.metadata_text, seg.suffix))
            trunc = {}
            for b in (base - 1, base, base + 1, base + 2, base + 3, base + 30, 300, 2048):
                try:
                    trunc[str(b)] = corpus.truncate_description(seg, b, vocab).full_prompt()
                except corpus.PromptBudgetError as e:
                    trunc[str(b)] = {"error": str(e)}
            assembly.append({"query": asdict(q), "item": asdict(it), "segments": asdict(seg),
                             "truncated": trunc})
    spans = [[t, [list(x) for x in tokenizer.encode_with_spans(t, vocab)]] for t in fuzz[:100] + prompt_texts[:2]]
    golden = {
        "assembly": assembly,
        "spans": spans,
        "texts": [[t, enc(t)] for t in fuzz + prompt_texts],
        "generator": "tests/golden/make_golden.py (reference prefrank tokenizer.py + corpus.py)",
        "fnv": {"offset": tokenizer.FNV_OFFSET, "prime": tokenizer.FNV_PRIME,
                "fnv1a_64": {w: tokenizer.fnv1a_64(w.encode()) for w in ["rust", "engineer", "a", ""]}},
        "vocab": vocab.to_config(),
        "encode": {s: enc(s) for s in [corpus.SYSTEM_PREFIX, "<|ans|>", "yes", "no", "rust engineer", "",
                                       "Senior Rust Engineer, Berlin!"]},
        "word_id": {w: vocab.word_id(w) for w in ["rust", "python", "yes", "<|meta|>"]},
        "requests": requests,
        "truncate_300": {"len": len(trunc300), "ends_with": trunc300[-3:]},
        "budget_error": budget_err,
    }
    with open(OUT, "w") as f:
        json.dump(golden, f, separators=(",", ":"))
    print(f"wrote {OUT}: {len(requests)} requests, {sum(len(r['prompts']) for r in requests)} prompts")


if __name__ == "__main__":
    main()
