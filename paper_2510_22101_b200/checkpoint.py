"""PRLK weight checkpoints so real, pruned checkpoints drop into the device
path, not only seeded random-init weights.

Reference: "single binary file, little-endian, header (magic PRLK, version,
ModelConfig fields) followed by tensors in declaration order; config also dumpable as JSON", and
SPEC.md:713, "model_version = checkpoint content hash".  The spec leaves the header encoding open;
this module pins it:

    offset 0   b"PRLK"
    offset 4   u32 version (= 1)
    offset 8   u32 n = byte length of the header JSON (space-padded to a multiple of 4)
    offset 12  header JSON (utf-8): {"config": ModelConfig fields, "dtype": "f32", "tensors": [[name, [dims]], ...]}
    then       tensors in declaration order, little-endian float32, row-major, no padding:
               token_embedding; per layer W_q, W_k, W_v, W_o, W_up, W_gate, W_down, rms_attn, rms_mlp;
               final_norm; head

``model_version`` is the SHA-256 of the file bytes (it keys the score cache).
Loading streams one tensor at a time through a memory map, so multi-GB checkpoints never sit in
host memory twice.
"""

from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import asdict

import numpy as np

from .config import ModelConfig
from .weights import LayerWeights, Weights

MAGIC = b"PRLK"
VERSION = 1
# declaration order of the per-layer tensors
LAYER_ORDER = ("W_q", "W_k", "W_v", "W_o", "W_up", "W_gate", "W_down", "rms_attn", "rms_mlp")


def _tensor_list(w: Weights):
    out = [("token_embedding", w.token_embedding)]
    for l, lw in enumerate(w.layers):
        for name in LAYER_ORDER:
            out.append((f"layers.{l}.{name}", getattr(lw, name)))
    out += [("final_norm", w.final_norm), ("head", w.head)]
    return out


def save_checkpoint(weights: Weights, path: str) -> str:
    """Write ``weights`` as a PRLK file; returns its model_version."""
    tensors = _tensor_list(weights)
    header = {
        "config": asdict(weights.config), "dtype": "f32",
        "tensors": [[n, [int(x) for x in a.shape]] for n, a in tensors],
    }
    hb = json.dumps(header, sort_keys=True).encode("utf-8")
    hb += b" " * (-len(hb) % 4)   # tensors start 4-byte aligned
    h = hashlib.sha256()
    with open(path, "wb") as f:
        for chunk in (MAGIC, struct.pack("<II", VERSION, len(hb)), hb):
            f.write(chunk)
            h.update(chunk)
        for _, a in tensors:
            b = np.ascontiguousarray(a, dtype="<f4").tobytes()
            f.write(b)
            h.update(b)
    return h.hexdigest()


def read_header(path: str) -> tuple[ModelConfig, dict, int]:
    with open(path, "rb") as f:
        head = f.read(12)
        if len(head) < 12 or head[:4] != MAGIC:
            raise ValueError(f"{path}: not a PRLK checkpoint (bad magic)")
        version, n = struct.unpack("<II", head[4:])
        if version != VERSION:
            raise ValueError(f"{path}: unsupported PRLK version {version}")
        header = json.loads(f.read(n).decode("utf-8"))
    if header.get("dtype") != "f32":
        raise ValueError(f"{path}: unsupported tensor dtype {header.get('dtype')!r}")
    return ModelConfig(**header["config"]), header, 12 + n


def _iter_tensors(path: str):
    cfg, header, off = read_header(path)
    mm = np.memmap(path, dtype="<f4", mode="r")
    if off % 4:
        raise ValueError(f"{path}: corrupt header length")
    pos = off // 4
    for name, shape in header["tensors"]:
        n = int(np.prod(shape))
        if pos + n > mm.size:
            raise ValueError(f"{path}: truncated at tensor {name}")
        a = np.asarray(mm[pos:pos + n]).reshape(shape)
        pos += n
        yield name, a
    if pos != mm.size:
        raise ValueError(f"{path}: {4 * (mm.size - pos)} trailing bytes")


def load_checkpoint(path: str) -> Weights:
    cfg, header, _ = read_header(path)
    _check_header(path, cfg, header)
    ts = dict(_iter_tensors(path))
    layers = []
    for l in range(cfg.n_layers):
        layers.append(LayerWeights(**{n: np.array(ts[f"layers.{l}.{n}"], dtype=np.float32) for n in LAYER_ORDER}))
    w = Weights(cfg, np.array(ts["token_embedding"], dtype=np.float32), layers,
                np.array(ts["final_norm"], dtype=np.float32), np.array(ts["head"], dtype=np.float32))
    _check_shapes(w)
    return w


def _check_shapes(w: Weights) -> None:
    """Shape discipline: every tensor's shape is a function of ModelConfig."""
    from .weights import layer_shapes

    cfg = w.config
    if w.token_embedding.shape != (cfg.vocab_size, cfg.d_model) or w.head.shape != (cfg.d_model, cfg.vocab_size):
        raise ValueError("checkpoint: embedding/head shape does not match ModelConfig")
    shapes = layer_shapes(cfg)
    for l, lw in enumerate(w.layers):
        for n, shp in shapes.items():
            if getattr(lw, n).shape != shp:
                raise ValueError(f"checkpoint: layer {l} {n} has shape {getattr(lw, n).shape}, expected {shp}")


def model_version(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 24), b""):
            h.update(chunk)
    return h.hexdigest()


def expected_tensors(cfg: ModelConfig) -> list[tuple[str, tuple[int, ...]]]:
    """Names and shapes of a PRLK file's tensors, in declaration order, as functions of the config
    (SPEC.md:222 shape discipline)."""
    from .weights import layer_shapes

    shapes = {**layer_shapes(cfg), "rms_attn": (cfg.d_model,), "rms_mlp": (cfg.d_model,)}
    out = [("token_embedding", (cfg.vocab_size, cfg.d_model))]
    for l in range(cfg.n_layers):
        out += [(f"layers.{l}.{n}", shapes[n]) for n in LAYER_ORDER]
    out += [("final_norm", (cfg.d_model,)), ("head", (cfg.d_model, cfg.vocab_size))]
    return out


def _check_header(path: str, cfg: ModelConfig, header: dict) -> None:
    got = [(str(n), tuple(int(x) for x in shp)) for n, shp in header.get("tensors", [])]
    want = expected_tensors(cfg)
    if got != want:
        bad = next((i for i, (a, b) in enumerate(zip(got, want)) if a != b), min(len(got), len(want)))
        g = got[bad] if bad < len(got) else "<missing>"
        w = want[bad] if bad < len(want) else "<none>"
        raise ValueError(f"{path}: tensor {bad} is {g}, the config requires {w} "
                         f"({len(got)} tensors listed, {len(want)} expected)")


def load_checkpoint_to_device(path: str, device="cuda"):
    """PRLK -> DeviceWeights, one layer at a time (the device layout of weights.to_device).  The
    header's tensor list is checked against the config (names, order, shapes, n_layers layers)
    before anything is uploaded, so the device never builds tensor maps over short buffers."""
    from .weights import DeviceWeights, _finish, _to_device_layer
    import torch

    cfg, header, _ = read_header(path)
    _check_header(path, cfg, header)
    dw = DeviceWeights(cfg, None, [], [], [], [], [], [], None, None, None, None, None)
    cur: dict = {}
    final = None
    for name, a in _iter_tensors(path):
        if name == "token_embedding":
            dw.embedding = torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=torch.bfloat16)
        elif name == "final_norm":
            final = np.array(a, dtype=np.float32)
        elif name == "head":
            _finish(dw, cfg, final, np.asarray(a), device)
        else:
            _, l, n = name.split(".")
            cur[n] = np.array(a, dtype=np.float32)
            if n == LAYER_ORDER[-1]:
                q, o, gu, dn = _to_device_layer(cfg, cur, device, cur["rms_attn"], cur["rms_mlp"])
                dw.w_qkv.append(q); dw.w_o.append(o); dw.w_gu.append(gu); dw.w_down.append(dn)
                dw.ln_attn.append(torch.from_numpy(cur["rms_attn"]).to(device))
                dw.ln_mlp.append(torch.from_numpy(cur["rms_mlp"]).to(device))
                cur = {}
    if len(dw.w_qkv) != cfg.n_layers or dw.w_yes is None:
        raise ValueError(f"{path}: loaded {len(dw.w_qkv)} of {cfg.n_layers} layers")
    return dw
