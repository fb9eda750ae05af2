"""Oracle restatement of the reference tokenizer (/root/reference/pkg/src/prefrank/tokenizer.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pure Python, written as an explicit
left-to-right scanner rather than the reference's regex:
* ids: specials "yes" -> 1, "no" -> 2, the nine template tags -> 3..11 in tag order
  (tokenizer.py:27-37, :60-64); any other word -> reserved + FNV-1a-64(utf-8) mod (size - reserved)
  (tokenizer.py:22-23, :72-76); Vocab(size=32768, reserved=16) by default (tokenizer.py:49-58).
* scan (tokenizer.py:98-134): the text is lowercased with str.lower(); at each position the tags
  are tried longest first, then a maximal [a-z0-9]+ run; anything else is skipped one character.
  Spans are (start, end) in the lowercased string (tokenizer.py:104-116).
Pinned by tests/test_tokenizer_oracle.py against the reference-generated golden vectors.
"""

from __future__ import annotations

FNV_OFFSET = 14695981039346656037
FNV_PRIME = 1099511628211
TAGS = ("<|sys|>", "<|/sys|>", "<|q|>", "<|/q|>", "<|meta|>", "<|/meta|>", "<|desc|>", "<|/desc|>", "<|ans|>")


def fnv1a_64(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h = ((h ^ b) * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def word_id(word: str, size: int = 32768, reserved: int = 16) -> int:
    if word == "yes":
        return 1
    if word == "no":
        return 2
    if word in TAGS:
        return 3 + TAGS.index(word)
    return reserved + fnv1a_64(word.encode("utf-8")) % (size - reserved)


def _is_word_char(c: str) -> bool:
    return ("a" <= c <= "z") or ("0" <= c <= "9")


def encode_with_spans(text: str, size: int = 32768, reserved: int = 16):
    s = text.lower()
    tags = sorted(TAGS, key=len, reverse=True)
    out, i, n = [], 0, len(s)
    while i < n:
        tag = next((t for t in tags if s.startswith(t, i)), None)
        if tag is not None:
            out.append((word_id(tag, size, reserved), i, i + len(tag)))
            i += len(tag)
        elif _is_word_char(s[i]):
            j = i
            while j < n and _is_word_char(s[j]):
                j += 1
            out.append((word_id(s[i:j], size, reserved), i, j))
            i = j
        else:
            i += 1
    return out


def encode(text: str, size: int = 32768, reserved: int = 16) -> list[int]:
    return [t for t, _, _ in encode_with_spans(text, size, reserved)]
