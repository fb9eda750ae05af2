"""PRLK checkpoint round trip and content-hash model_version."""

import numpy as np
import pytest

from paper_2510_22101_b200 import CONFIGS, init_weights
from paper_2510_22101_b200.checkpoint import (load_checkpoint, model_version, read_header,
                                             save_checkpoint)
from paper_2510_22101_b200.pruning import PruneRecipe, apply_recipe


def test_round_trip_bitwise(tmp_path):
    cfg = CONFIGS["TINY_GQA"]
    w = init_weights(cfg, 3)
    w.layers[1].rms_mlp = np.linspace(0.5, 1.5, cfg.d_model).astype(np.float32)
    p = tmp_path / "m.prlk"
    v = save_checkpoint(w, str(p))
    assert v == model_version(str(p)) and len(v) == 64
    r = load_checkpoint(str(p))
    assert r.config == cfg
    assert np.array_equal(r.token_embedding, w.token_embedding) and np.array_equal(r.head, w.head)
    for a, b in zip(r.layers, w.layers):
        for f in ("W_q", "W_k", "W_v", "W_o", "W_up", "W_gate", "W_down", "rms_attn", "rms_mlp"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
    cfg2, header, _ = read_header(str(p))
    assert cfg2 == cfg and header["tensors"][0] == ["token_embedding", [cfg.vocab_size, cfg.d_model]]


def test_version_changes_with_weights_and_pruned_shapes(tmp_path):
    cfg = CONFIGS["TINY_GQA"]
    w = init_weights(cfg, 0)
    v1 = save_checkpoint(w, str(tmp_path / "a.prlk"))
    w.layers[0].W_down[3, 7] += 1.0
    v2 = save_checkpoint(w, str(tmp_path / "b.prlk"))
    assert v1 != v2
    pw = apply_recipe(w, PruneRecipe(mlp_sparsity=0.4, layers_to_remove=(2,), kv_groups_to_keep=1))
    save_checkpoint(pw, str(tmp_path / "c.prlk"))
    r = load_checkpoint(str(tmp_path / "c.prlk"))
    assert (r.config.d_ff, r.config.n_layers, r.config.n_heads) == (360, 2, 2)
    assert r.param_count() == pw.param_count()


def test_rejects_corrupt_files(tmp_path):
    p = tmp_path / "x.prlk"
    p.write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(ValueError):
        load_checkpoint(str(p))
    w = init_weights(CONFIGS["TINY"], 0)
    good = tmp_path / "g.prlk"
    save_checkpoint(w, str(good))
    data = good.read_bytes()
    (tmp_path / "t.prlk").write_bytes(data[:-8])
    with pytest.raises(ValueError):
        load_checkpoint(str(tmp_path / "t.prlk"))


def _rewrite_header(src, dst, edit):
    """Copy a PRLK file with its header JSON edited (tensor bytes unchanged)."""
    import json
    import struct

    data = open(src, "rb").read()
    n = struct.unpack("<I", data[8:12])[0]
    header = json.loads(data[12:12 + n])
    edit(header)
    hb = json.dumps(header, sort_keys=True).encode()
    hb += b" " * (-len(hb) % 4)
    open(dst, "wb").write(data[:4] + struct.pack("<II", 1, len(hb)) + hb + data[12 + n:])


def test_header_tensor_list_must_match_config(tmp_path):
    """the device loader trusted the header's tensor list.  A checkpoint whose
    list omits a layer or disagrees with the config's shapes is rejected before any upload."""
    from paper_2510_22101_b200.checkpoint import expected_tensors

    cfg = CONFIGS["TINY_GQA"]
    good = str(tmp_path / "g.prlk")
    save_checkpoint(init_weights(cfg, 0), good)
    assert [(n, tuple(s)) for n, s in read_header(good)[1]["tensors"]] == expected_tensors(cfg)
    # claims one layer more than it holds
    _rewrite_header(good, tmp_path / "a.prlk", lambda h: h["config"].update(n_layers=cfg.n_layers + 1))
    # a layer's W_o listed with a smaller shape (same element count elsewhere would go unnoticed)
    def shrink(h):
        for t in h["tensors"]:
            if t[0] == "layers.1.W_o":
                t[1] = [t[1][0] // 2, t[1][1] * 2]
    _rewrite_header(good, tmp_path / "b.prlk", shrink)
    # the last layer's tensors dropped from the list
    _rewrite_header(good, tmp_path / "c.prlk",
                    lambda h: h.update(tensors=[t for t in h["tensors"] if not t[0].startswith("layers.2.")]))
    for bad in ("a", "b", "c"):
        with pytest.raises(ValueError):
            load_checkpoint(str(tmp_path / f"{bad}.prlk"))
        try:
            import torch  # noqa: F401
            from paper_2510_22101_b200.checkpoint import load_checkpoint_to_device
        except ImportError:
            continue
        with pytest.raises(ValueError):
            load_checkpoint_to_device(str(tmp_path / f"{bad}.prlk"), device="cpu")
