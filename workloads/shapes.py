"""Tensor inventories of the paper's workloads (no checkpoint arithmetic here).

Shapes follow the GPT-3 family the paper evaluates (§5.2, Table
`tb:gpt-setup`; architecture "based on GPT-3") in the
Megatron layout (fused QKV, 4x MLP), vocabulary padded to 50304, sequence
2048. The checkpoint state is mixed-precision Adam: 16-bit params,
fp32 master params, fp32 momentum and variance; the default profile `adam16`
also keeps bf16 grads (ZeRO's 2+2+12 accounting, BASELINE.json configs
"~21/~107/~208 GB" = 16 B/param), `adam14` is the paper's 2+4+4+4.

Configs C1..C5 are BASELINE.json `configs[0..4]`.
"""
from __future__ import annotations

from dataclasses import dataclass, field

SECTIONS = ("param", "grad", "master", "exp_avg", "exp_avg_sq")
SECTION_DTYPE = {"param": "bf16", "grad": "bf16", "master": "f32",
                 "exp_avg": "f32", "exp_avg_sq": "f32"}
ITEMSIZE = {"f32": 4, "bf16": 2, "f16": 2, "f64": 8, "i64": 8, "i32": 4, "u8": 1}

VOCAB = 50304
SEQ = 2048


@dataclass(frozen=True)
class Spec:
    """One checkpointed tensor: name, shape, dtype, section, owner.

    owner = -1: replicated on every DP rank ("DP ranks hold identical
    checkpoint data"); owner = r: rank r's own partition (ZeRO / experts).
    gen/gen_id drive the seeded generator (workloads.gen); a `param` tensor
    is bf16(master) of the same model tensor, so it shares the master gen_id.
    """
    name: str
    shape: tuple
    dtype: str
    section: str
    owner: int = -1
    gen: str = "randn"
    gen_id: int = 0

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= int(s)
        return n

    @property
    def nbytes(self) -> int:
        return self.numel * ITEMSIZE[self.dtype]


# ----------------------------------------------------------------------------
# model tensor lists (state-dict order)
# ----------------------------------------------------------------------------
def gpt3_tensors(d: int, layers: int, vocab: int = VOCAB, seq: int = SEQ):
    """Megatron GPT-3 parameter list [(name, shape)] in state-dict order.

    Per layer 12*d^2 + 13*d parameters; plus word/position embeddings and the
    final LayerNorm. Reproduces 1.3B = 1,315,819,520 (d=2048, L=24)."""
    out = [("word_embeddings.weight", (vocab, d)),
           ("position_embeddings.weight", (seq, d))]
    for i in range(layers):
        p = f"layers.{i}."
        out += [
            (p + "input_layernorm.weight", (d,)),
            (p + "input_layernorm.bias", (d,)),
            (p + "attention.query_key_value.weight", (3 * d, d)),
            (p + "attention.query_key_value.bias", (3 * d,)),
            (p + "attention.dense.weight", (d, d)),
            (p + "attention.dense.bias", (d,)),
            (p + "post_attention_layernorm.weight", (d,)),
            (p + "post_attention_layernorm.bias", (d,)),
            (p + "mlp.dense_h_to_4h.weight", (4 * d, d)),
            (p + "mlp.dense_h_to_4h.bias", (4 * d,)),
            (p + "mlp.dense_4h_to_h.weight", (d, 4 * d)),
            (p + "mlp.dense_4h_to_h.bias", (d,)),
        ]
    out += [("final_layernorm.weight", (d,)), ("final_layernorm.bias", (d,))]
    return out


def gpt3_param_count(d: int, layers: int, vocab: int = VOCAB, seq: int = SEQ) -> int:
    return layers * (12 * d * d + 13 * d) + vocab * d + seq * d + 2 * d


def moe_tensors(d: int = 2048, layers: int = 24, experts: int = 64,
                vocab: int = VOCAB, seq: int = SEQ):
    """MoE GPT (1.3B base, MoE FFN in every layer, `experts` experts).

    Returns (replicated [(name, shape)], expert [(layer, expert, name, shape)]).
    Each expert is one FFN (W1 [4d,d], b1 [4d], W2 [d,4d], b2 [d]); the gate
    [experts, d] is replicated. 64 experts x 24 layers gives ~52.07B params
    (BASELINE.json configs[4], "~50B")."""
    rep = [("word_embeddings.weight", (vocab, d)),
           ("position_embeddings.weight", (seq, d))]
    exp = []
    for i in range(layers):
        p = f"layers.{i}."
        rep += [
            (p + "input_layernorm.weight", (d,)),
            (p + "input_layernorm.bias", (d,)),
            (p + "attention.query_key_value.weight", (3 * d, d)),
            (p + "attention.query_key_value.bias", (3 * d,)),
            (p + "attention.dense.weight", (d, d)),
            (p + "attention.dense.bias", (d,)),
            (p + "post_attention_layernorm.weight", (d,)),
            (p + "post_attention_layernorm.bias", (d,)),
            (p + "mlp.gate.weight", (experts, d)),
        ]
        for e in range(experts):
            q = f"{p}mlp.experts.{e}."
            exp += [(i, e, q + "dense_h_to_4h.weight", (4 * d, d)),
                    (i, e, q + "dense_h_to_4h.bias", (4 * d,)),
                    (i, e, q + "dense_4h_to_h.weight", (d, 4 * d)),
                    (i, e, q + "dense_4h_to_h.bias", (d,))]
    rep += [("final_layernorm.weight", (d,)), ("final_layernorm.bias", (d,))]
    return rep, exp


def tiny_tensors():
    """C1: 8 random fp32/bf16 tensors totalling ~64 MB (67,104,188 data bytes).

    Chosen to exercise the ragged cases: a bf16 row of odd length, a tensor
    whose byte size is 14 mod 16 (vector tail), a 7-element tensor and a
    0-dim scalar."""
    return [
        ("t0", (4096, 1024), "f32"),
        ("t1", (4096, 2048), "bf16"),
        ("t2", (2048, 1024), "f32"),
        ("t3", (2048, 2047), "bf16"),
        ("t4", (1000, 2097), "f32"),
        ("t5", (3, 1398101), "bf16"),
        ("t6", (7,), "f32"),
        ("t7", (), "bf16"),
    ]


# ----------------------------------------------------------------------------
# configs -> per-rank Spec lists
# ----------------------------------------------------------------------------
def _adam_specs(params, profile: str, owner: int = -1, prefix: str = "",
                gen_base: int = 0):
    """Section-major Adam state: all params, then grads, master, m, v."""
    secs = SECTIONS if profile == "adam16" else tuple(s for s in SECTIONS if s != "grad")
    out = []
    for sec in secs:
        for j, (name, shape) in enumerate(params):
            gid = gen_base + j if sec in ("param", "master") else \
                gen_base + j + (SECTIONS.index(sec) << 24)
            out.append(Spec(f"{sec}/{prefix}{name}", tuple(shape),
                            SECTION_DTYPE[sec], sec, owner, sec, gid))
    return out


CONFIGS = {
    # name: (description, builder kwargs)
    "c1_tiny": "C1: tiny state dict, 8 random fp32/bf16 tensors, ~64 MB, 1 rank",
    "c2_gpt3_1.3b": "C2: GPT-3 1.3B dense mixed-precision Adam state (~21 GB), replicated",
    "c3_gpt3_6.7b": "C3: GPT-3 6.7B dense mixed-precision Adam state (~107 GB), replicated",
    "c4_gpt3_13b_zero": "C4: GPT-3 13B, ZeRO-partitioned state (~208 GB over k ranks), rank-local",
    "c5_moe_64e": "C5: MoE GPT 1.3B base x 64 experts (~52B params), expert-sharded at EP=k",
    # small variants used by the parity tests (same structure, seconds to check)
    "gpt3_small": "GPT-3 structure d=256 L=2 (test size)",
    "gpt3_odd": "GPT-3 structure d=320 L=2, vocab 1000 (rows not page multiples: padding)",
    "zero_small": "ZeRO-partitioned GPT-3 d=256 L=2 (test size, rank-local)",
    "moe_small": "MoE GPT d=128 L=2, 8 experts (test size, replicated + rank-local)",
}


def config_specs(cfg: str, rank: int = 0, k: int = 1, profile: str = "adam16"):
    """Ordered Spec list that DP rank `rank` of `k` checkpoints for `cfg`."""
    if cfg == "c1_tiny":
        return [Spec(n, s, dt, "other", -1, "randn", i)
                for i, (n, s, dt) in enumerate(tiny_tensors())]
    dense = {"c2_gpt3_1.3b": (2048, 24, VOCAB), "c3_gpt3_6.7b": (4096, 32, VOCAB),
             "gpt3_small": (256, 2, VOCAB), "gpt3_odd": (320, 2, 1000)}
    if cfg in dense:
        d, L, v = dense[cfg]
        return _adam_specs(gpt3_tensors(d, L, v, SEQ if d > 320 else 256), profile)
    zero = {"c4_gpt3_13b_zero": (5120, 40, VOCAB), "zero_small": (256, 2, VOCAB)}
    if cfg in zero:
        d, L, v = zero[cfg]
        params = []
        for name, shape in gpt3_tensors(d, L, v, SEQ if d > 256 else 256):
            assert shape[0] % k == 0, (name, shape, k)
            params.append((name, (shape[0] // k,) + tuple(shape[1:])))
        return _adam_specs(params, profile, owner=rank, prefix=f"zero{rank}.",
                           gen_base=(rank + 1) * 1_000_003)
    moe = {"c5_moe_64e": (2048, 24, 64, VOCAB, SEQ), "moe_small": (128, 2, 8, 1000, 256)}
    if cfg in moe:
        d, L, E, v, s = moe[cfg]
        assert E % k == 0
        rep, exp = moe_tensors(d, L, E, v, s)
        mine = [(n, sh) for (_, e, n, sh) in exp if e // (E // k) == rank]
        return (_adam_specs(rep, profile) +
                _adam_specs(mine, profile, owner=rank,
                            gen_base=(rank + 1) * 1_000_003))
    raise KeyError(cfg)


def state_bytes(specs) -> int:
    return sum(s.nbytes for s in specs)
