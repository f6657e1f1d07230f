"""Synthetic parameter-group tables for the BASELINE.json configs.

Each table lists one group (= one reference ParamBlock) per model tensor, in
layer order; the update order is the reverse.  No weights are
loaded (no network): values come from the device seeded_fill.
"""
from __future__ import annotations


def bert_large_sizes() -> list[int]:
    """BERT-large (hidden 1024, 24 layers, FFN 4096, vocab 30522): 336,226,108
    params in 398 tensors — config 2 ("340M")."""
    H, L, FF, V, P, TV = 1024, 24, 4096, 30522, 512, 2
    s = [V * H, P * H, TV * H, H, H]                     # embeddings + LN
    for _ in range(L):
        s += [H * H, H] * 3                               # q, k, v
        s += [H * H, H, H, H]                             # attn out + LN
        s += [H * FF, FF, FF * H, H, H, H]                # FFN + LN
    s += [H * H, H]                                       # pooler
    s += [H * H, H, H, H, V]                              # MLM transform + LN + decoder bias
    s += [H * 2, 2]                                       # NSP
    return s


def gpt2_xl_sizes() -> list[int]:
    """GPT-2 XL (d 1600, 48 layers, vocab 50257, ctx 1024): 1,557,611,200
    params in 580 tensors — config 3."""
    D, L, V, P = 1600, 48, 50257, 1024
    s = [V * D, P * D]
    for _ in range(L):
        s += [D, D, D * 3 * D, 3 * D, D * D, D, D, D, D * 4 * D, 4 * D, 4 * D * D, D]
    s += [D, D]
    return s


def flat_sizes(total: int, groups: int) -> list[int]:
    """`total` params split into `groups` near-equal groups (config 1: 10M/100)."""
    base, rem = divmod(total, groups)
    return [base + (1 if i < rem else 0) for i in range(groups)]


def one_billion_sizes() -> list[int]:
    """The north_star 1B-parameter fp32 target: 1,000,000,000 params as 250
    groups of 4M (transformer-like tensor granularity)."""
    return flat_sizes(1_000_000_000, 250)


CONFIGS = {
    "sgdm10m": dict(sizes=lambda: flat_sizes(10_000_000, 100), desc="config 1: SGDM 10M flat, 100 groups"),
    "adam340m": dict(sizes=bert_large_sizes, desc="config 2: Adam BERT-large 336M, 398 groups"),
    "adam1b": dict(sizes=one_billion_sizes, desc="north_star target: Adam 1B fp32, 250 groups"),
    "gpt2xl": dict(sizes=gpt2_xl_sizes, desc="config 3: GPT-2 XL 1.56B, 580 groups"),
}
