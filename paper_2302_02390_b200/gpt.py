"""GPT-shaped parameter groups for the benchmark (SURVEY §8 / BASELINE.json configs).

Standard GPT-2/3 shapes (vocab 50,257, context 1,024, tied embeddings).  One
FSDP group per transformer block plus one root group (wte, wpe), as FSDP2 wraps
a GPT: the block group's dense tensors (attn qkv, attn proj, mlp fc, mlp proj)
are quantized; biases and LayerNorms travel in full precision and are not part
of the quantized buckets (sharded.py:359-371).
"""

from __future__ import annotations

from dataclasses import dataclass

GPT_CONFIGS = {
    "gpt2-125m": dict(d=768, layers=12, vocab=50257, ctx=1024),
    "gpt2-350m": dict(d=1024, layers=24, vocab=50257, ctx=1024),
    "gpt-1.3b": dict(d=2048, layers=24, vocab=50257, ctx=1024),
    "gpt-tiny": dict(d=128, layers=2, vocab=50257, ctx=1024),
}


@dataclass(frozen=True)
class ParamGroup:
    name: str
    tensors: tuple  # ((name, numel), ...) dense tensors of the group

    @property
    def numel(self) -> int:
        return sum(n for _, n in self.tensors)


def dense_groups(model: str):
    c = GPT_CONFIGS[model]
    d = c["d"]
    groups = [ParamGroup("root", (("wte", c["vocab"] * d), ("wpe", c["ctx"] * d)))]
    for i in range(c["layers"]):
        groups.append(ParamGroup(f"h{i}", ((f"h{i}.attn.c_attn", d * 3 * d), (f"h{i}.attn.c_proj", d * d),
                                           (f"h{i}.mlp.c_fc", d * 4 * d), (f"h{i}.mlp.c_proj", 4 * d * d))))
    return groups


def dense_numel(model: str) -> int:
    return sum(g.numel for g in dense_groups(model))
