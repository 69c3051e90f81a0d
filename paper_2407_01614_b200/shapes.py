"""Flat parameter-buffer shapes of the BASELINE.json workloads.

One flat buffer per ZeRO-3 module (decoder block, embedding, lm_head, final norm):
the module granularity of Alg. 1 (reading R23).  The paper names
the models only; the element counts are derived from the
public Hugging Face configs — see DESIGN.md §6.
"""
from __future__ import annotations


def _falcon7b():
    h, ffn = 4544, 18176
    qkv = h * (h + 2 * 64)            # 71 query heads + 1 shared K/V head (MQA), head_dim 64
    block = qkv + h * h + 2 * h * ffn + 2 * h   # attn qkv + dense + MLP up/down + 1 LN (w+b)
    return [65024 * h] + [block] * 32 + [2 * h]   # tied embedding, 32 blocks, ln_f (w+b)


def _llama(h, ffn, layers, kv_heads=None, heads=None, vocab=32000):
    if kv_heads is None:
        attn = 4 * h * h
    else:
        hd = h // heads
        attn = 2 * h * h + 2 * h * kv_heads * hd
    block = attn + 3 * h * ffn + 2 * h
    return [vocab * h] + [block] * layers + [h] + [vocab * h]   # embed, blocks, norm, lm_head


def _falcon40b():
    h, ffn, hd, kv = 8192, 32768, 64, 8
    qkv = h * (h + 2 * kv * hd)
    block = qkv + h * h + 2 * h * ffn + 4 * h      # 2 LNs (w+b)
    return [65024 * h] + [block] * 60 + [2 * h]


def _toy():
    d, hdim, o = 512, 1024, 512
    return [hdim * d + hdim, o * hdim + o]


MODELS = {
    "toy": _toy(),                                            # 1,050,112 (C1)
    "falcon7b": _falcon7b(),                                  # 6,921,720,704 (C2)
    "llama2_7b": _llama(4096, 11008, 32),                     # 6,738,415,616
    "llama2_13b": _llama(5120, 13824, 40),                    # 13,015,864,320 (C3)
    "falcon40b": _falcon40b(),                                # 41,303,293,952 (C4)
    "falcon40b_block": [_falcon40b()[1]],                     # one decoder block, per-layer timing (C4)
    "falcon7b_block": [_falcon7b()[1]],                       # one C2 decoder block (ncu captures of the bench's launches)
    "llama2_70b_layers": [_llama(8192, 28672, 1, kv_heads=8, heads=64)[1]] * 4,   # 4 x 855,654,400 (C5)
}

PARAM_DTYPE = {"toy": "f32"}   # everything else: bf16 params + fp32 master/Adam (R9)


def numels(model: str) -> list[int]:
    return list(MODELS[model])


def total(model: str) -> int:
    return sum(MODELS[model])
