"""Synthetic graphs of the BASELINE.json config shapes, emitted as the
reference's Graph Interchange documents (reference SPEC.md:552).

The reference ships only toy generators (pkg/src/memplan/graphgen.py:202-279);
the configs the benchmark names -- a seeded layered DAG, GPT-2 small, BERT-large
and GPT2-XL training graphs -- do not exist there, so they are built here:

* ``layered_dag_doc``: SURVEY §6 rules (layers x width ops, k outputs per op,
  every previous-layer tensor gets >= 1 next-layer consumer plus an extra one
  with probability p, every op reads >= 1 previous-layer tensor, sizes
  ``randint(lo, hi)`` MB from ``random.Random(seed)``).
* ``transformer_training_doc``: an FX-granularity forward pass (layer norms as
  mean/var/normalize/affine, q/k/v views and permutes, tanh-GELU as its
  elementwise ops, dropout masks), an autograd-style mirrored backward pass
  with separate dgrad/wgrad ops per matmul, gradient accumulation ops where a
  tensor fans out, and the reference's 4-op Adam branch per parameter
  gradient (graphgen.py:63-74, names ``adam.m{k}`` ... so the planner's alpha
  resolution by name prefix, ordering.py:289-307, sees "adam").

Byte sizes are element counts x dtype bytes (fp32 activations, 1-byte dropout
masks), so all arithmetic is integer and exact.
"""

from __future__ import annotations

import hashlib
import json
import random
from dataclasses import dataclass

MB = 1 << 20


# ---------------------------------------------------------------- layered DAG

def layered_dag_doc(layers: int = 50, width: int = 20, outs_per_op: int = 3,
                    extra_p: float = 0.3, size_range_mb: tuple[int, int] = (1, 64),
                    seed: int = 0) -> dict:
    rng = random.Random(seed)
    lo, hi = size_range_mb
    ops: list[dict] = []
    tensors: list[dict] = []
    prev_tensors: list[int] = []
    for L in range(layers):
        layer_ops = list(range(len(ops), len(ops) + width))
        inputs: dict[int, set[int]] = {v: set() for v in layer_ops}
        if L > 0:
            for t in prev_tensors:
                inputs[rng.choice(layer_ops)].add(t)
                if rng.random() < extra_p:
                    inputs[rng.choice(layer_ops)].add(t)
            for v in layer_ops:
                if not inputs[v]:
                    inputs[v].add(rng.choice(prev_tensors))
        cur: list[int] = []
        for v in layer_ops:
            outs = []
            for _ in range(outs_per_op):
                tid = len(tensors)
                tensors.append({"id": tid, "size_bytes": rng.randint(lo, hi) * MB})
                outs.append(tid)
            cur.extend(outs)
            ops.append({"id": v, "name": f"l{L}.op{v - layer_ops[0]}", "kind": "forward",
                        "inputs": sorted(inputs[v]), "outputs": outs})
        prev_tensors = cur
    return {"ops": ops, "tensors": tensors}


# ------------------------------------------------------- transformer training

@dataclass(frozen=True)
class TransformerShape:
    name: str
    layers: int
    d_model: int
    heads: int
    seq: int
    batch: int
    vocab: int
    decoder: bool          # GPT (pre-LN, causal mask, tanh GELU) vs BERT (post-LN, erf GELU)
    traced: bool = False   # op granularity of a traced eager training step: LayerNorm as its
                           # aten decomposition, Adam's per-parameter update unfused


GPT2_SMALL = TransformerShape("gpt2-small", 12, 768, 12, 1024, 8, 50257, True)
BERT_LARGE = TransformerShape("bert-large", 24, 1024, 16, 512, 8, 30522, False)
# GPT2-XL at the paper's granularity (">10 thousand operators"):
# 11,217 ops / 10,782 tensors
GPT2_XL = TransformerShape("gpt2-xl", 48, 1600, 25, 1024, 1, 50257, True, traced=True)
SHAPES = {s.name: s for s in (GPT2_SMALL, BERT_LARGE, GPT2_XL)}


class _Builder:
    """Forward tape + reverse-mode expansion into interchange ops."""

    def __init__(self) -> None:
        self.ops: list[dict] = []
        self.sizes: list[int] = []
        self.tape: list[tuple] = []     # (name, inputs, outputs, rule)
        self.params: list[tuple[str, int]] = []

    def tensor(self, nbytes: int) -> int:
        self.sizes.append(int(nbytes))
        return len(self.sizes) - 1

    def emit(self, name: str, kind: str, inputs: list[int], outputs: list[int]) -> int:
        self.ops.append({"id": len(self.ops), "name": name, "kind": kind,
                         "inputs": list(inputs), "outputs": list(outputs)})
        return len(self.ops) - 1

    # forward op with a backward rule:
    #   rule = list of (grad_target, extra_inputs) where grad_target is an input
    #   index (gradient of that input) or ("param", nbytes) for a weight grad;
    #   extra_inputs are saved forward tensors the backward op reads.
    def fwd(self, name: str, inputs: list[int], out_bytes: list[int], rule=(), kind="forward") -> list[int]:
        outs = [self.tensor(b) for b in out_bytes]
        self.emit(name, kind, inputs, outs)
        self.tape.append((name, list(inputs), outs, list(rule)))
        return outs

    def backward(self, loss_grad_of: int, seed_bytes: int) -> None:
        grads: dict[int, list[int]] = {}
        seed = self.tensor(seed_bytes)
        # the loss op itself emitted the seed gradient
        self.ops[-1]["outputs"].append(seed)
        grads[loss_grad_of] = [seed]
        param_k = 0
        for name, inputs, outs, rule in reversed(self.tape):
            gouts = []
            for o in outs:
                gs = grads.pop(o, None)
                if not gs:
                    continue
                if len(gs) > 1:  # fan-out: accumulate contributions
                    acc = self.tensor(self.sizes[o])
                    self.emit(f"{name}.grad_acc", "backward", gs, [acc])
                    gs = [acc]
                gouts.append(gs[0])
            if not gouts:
                continue
            def resolve(i):
                return inputs[i] if isinstance(i, int) else outs[i[1]]

            for target, saved in rule:
                if isinstance(target, tuple):          # weight gradient
                    tag, nbytes = target
                    gw = self.tensor(nbytes)
                    self.emit(f"{name}.{tag}_wgrad", "backward", gouts + [resolve(i) for i in saved], [gw])
                    self.params.append((f"{name}.{tag}", gw))
                    param_k += 1
                else:
                    x = inputs[target]
                    gx = self.tensor(self.sizes[x])
                    suffix = "dgrad" if len(rule) > 1 else "bwd"
                    self.emit(f"{name}.{suffix}{target}", "backward",
                              gouts + [resolve(i) for i in saved], [gx])
                    grads.setdefault(x, []).append(gx)

    def adam(self, traced: bool = False) -> None:
        if traced:
            # torch.optim.Adam (foreach=False) as traced per parameter:
            # exp_avg.mul_(b1).add_(g, alpha=1-b1); exp_avg_sq.mul_(b2).addcmul_(g, g,
            # value=1-b2); denom = (exp_avg_sq.sqrt() / bc2_sqrt).add_(eps);
            # param.addcdiv_(exp_avg, denom, value=-step_size)
            for k, (_pname, gw) in enumerate(self.params):
                sz = self.sizes[gw]
                m1, m2, v1, v2, sq, dn, de = (self.tensor(sz) for _ in range(7))
                self.emit(f"adam.m_mul{k}", "weight_update", [gw], [m1])
                self.emit(f"adam.m_add{k}", "weight_update", [m1, gw], [m2])
                self.emit(f"adam.v_mul{k}", "weight_update", [gw], [v1])
                self.emit(f"adam.v_addcmul{k}", "weight_update", [v1, gw], [v2])
                self.emit(f"adam.sqrt{k}", "weight_update", [v2], [sq])
                self.emit(f"adam.div{k}", "weight_update", [sq], [dn])
                self.emit(f"adam.add_eps{k}", "weight_update", [dn], [de])
                self.emit(f"adam.addcdiv{k}", "weight_update", [m2, de], [])
            return
        # one 4-op branch per parameter gradient, reference graphgen.py:63-74
        for k, (_pname, gw) in enumerate(self.params):
            sz = self.sizes[gw]
            mo, vo, st = self.tensor(sz), self.tensor(sz), self.tensor(sz)
            self.emit(f"adam.m{k}", "weight_update", [gw], [mo])
            self.emit(f"adam.v{k}", "weight_update", [gw], [vo])
            self.emit(f"adam.step{k}", "weight_update", [mo, vo], [st])
            self.emit(f"adam.apply{k}", "weight_update", [st], [])

    def doc(self) -> dict:
        return {"ops": self.ops,
                "tensors": [{"id": i, "size_bytes": s} for i, s in enumerate(self.sizes)]}


def transformer_training_doc(shape: TransformerShape) -> dict:
    B, S, D, H, V = shape.batch, shape.seq, shape.d_model, shape.heads, shape.vocab
    F = 4 * D
    f4 = 4
    act = B * S * D * f4
    b = _Builder()
    OUT = lambda i: ("out", i)  # noqa: E731  saved forward output reference

    tokens = b.fwd("data.tokens", [], [B * S * 8], kind="forward")[0]
    labels = b.fwd("data.labels", [], [B * S * 8], kind="forward")[0]
    wte = b.fwd("embed.wte", [tokens], [act], rule=[(("W", V * D * f4), [0])])[0]
    wpe = b.fwd("embed.wpe", [tokens], [act], rule=[(("W", S * D * f4), [0])])[0]
    x = b.fwd("embed.add", [wte, wpe], [act], rule=[(0, []), (1, [])])[0]

    def layer_norm(pfx: str, x: int) -> int:
        if shape.traced:   # aten decomposition of native_layer_norm
            mu = b.fwd(f"{pfx}.mean", [x], [B * S * f4], rule=[(0, [])])[0]
            xc = b.fwd(f"{pfx}.sub", [x, mu], [act], rule=[(0, []), (1, [])])[0]
            sq = b.fwd(f"{pfx}.pow", [xc], [act], rule=[(0, [0])])[0]
            var = b.fwd(f"{pfx}.var", [sq], [B * S * f4], rule=[(0, [])])[0]
            ve = b.fwd(f"{pfx}.add_eps", [var], [B * S * f4], rule=[(0, [])])[0]
            rs = b.fwd(f"{pfx}.rsqrt", [ve], [B * S * f4], rule=[(0, [OUT(0)])])[0]
            xhat = b.fwd(f"{pfx}.mul", [xc, rs], [act], rule=[(0, [1]), (1, [0])])[0]
            y = b.fwd(f"{pfx}.mul_gamma", [xhat], [act], rule=[(("gamma", D * f4), [0]), (0, [])])[0]
            return b.fwd(f"{pfx}.add_beta", [y], [act], rule=[(("beta", D * f4), []), (0, [])])[0]
        mu = b.fwd(f"{pfx}.mean", [x], [B * S * f4], rule=[(0, [])])[0]
        var = b.fwd(f"{pfx}.var", [x, mu], [B * S * f4], rule=[(0, [0, 1])])[0]
        xhat = b.fwd(f"{pfx}.normalize", [x, mu, var], [act], rule=[(0, [OUT(0), 2])])[0]
        return b.fwd(f"{pfx}.affine", [xhat], [act],
                     rule=[(("gamma", D * f4), [0]), (("beta", D * f4), []), (0, [])])[0]

    def linear(pfx: str, x: int, d_in: int, d_out: int, rows: int = B * S) -> int:
        y = b.fwd(f"{pfx}.mm", [x], [rows * d_out * f4], rule=[(("W", d_in * d_out * f4), [0]), (0, [])])[0]
        return b.fwd(f"{pfx}.bias", [y], [rows * d_out * f4], rule=[(("b", d_out * f4), []), (0, [])])[0]

    def dropout(pfx: str, x: int, nelem: int) -> int:
        y, _mask = b.fwd(f"{pfx}.dropout", [x], [nelem * f4, nelem], rule=[(0, [OUT(1)])])
        return y

    def gelu(pfx: str, x: int) -> int:
        n = B * S * F
        if shape.decoder:  # tanh approximation as traced: x^3, fma, tanh, 1+, x*, *0.5
            c = b.fwd(f"{pfx}.pow3", [x], [n * f4], rule=[(0, [0])])[0]
            u = b.fwd(f"{pfx}.fma", [x, c], [n * f4], rule=[(0, []), (1, [])])[0]
            th = b.fwd(f"{pfx}.tanh", [u], [n * f4], rule=[(0, [OUT(0)])])[0]
            one = b.fwd(f"{pfx}.add1", [th], [n * f4], rule=[(0, [])])[0]
            xm = b.fwd(f"{pfx}.mulx", [x, one], [n * f4], rule=[(0, [1]), (1, [0])])[0]
            return b.fwd(f"{pfx}.half", [xm], [n * f4], rule=[(0, [])])[0]
        e = b.fwd(f"{pfx}.erf", [x], [n * f4], rule=[(0, [0])])[0]
        one = b.fwd(f"{pfx}.add1", [e], [n * f4], rule=[(0, [])])[0]
        xm = b.fwd(f"{pfx}.mulx", [x, one], [n * f4], rule=[(0, [1]), (1, [0])])[0]
        return b.fwd(f"{pfx}.half", [xm], [n * f4], rule=[(0, [])])[0]

    def attention(pfx: str, h: int) -> int:
        qkv = linear(f"{pfx}.qkv", h, D, 3 * D)
        heads = []
        for nm in ("q", "k", "v"):
            sl = b.fwd(f"{pfx}.split_{nm}", [qkv], [act], rule=[(0, [])])[0]
            vw = b.fwd(f"{pfx}.view_{nm}", [sl], [act], rule=[(0, [])])[0]
            heads.append(b.fwd(f"{pfx}.permute_{nm}", [vw], [act], rule=[(0, [])])[0])
        q, k, v = heads
        kt = b.fwd(f"{pfx}.transpose_k", [k], [act], rule=[(0, [])])[0]
        sc_n = B * H * S * S
        s = b.fwd(f"{pfx}.scores", [q, kt], [sc_n * f4], rule=[(0, [1]), (1, [0])])[0]
        s = b.fwd(f"{pfx}.scale", [s], [sc_n * f4], rule=[(0, [])])[0]
        s = b.fwd(f"{pfx}.mask", [s], [sc_n * f4], rule=[(0, [])])[0]
        p = b.fwd(f"{pfx}.softmax", [s], [sc_n * f4], rule=[(0, [OUT(0)])])[0]
        p = dropout(f"{pfx}.attn", p, sc_n)
        ctx = b.fwd(f"{pfx}.context", [p, v], [act], rule=[(0, [1]), (1, [0])])[0]
        ctx = b.fwd(f"{pfx}.permute_ctx", [ctx], [act], rule=[(0, [])])[0]
        ctx = b.fwd(f"{pfx}.merge_heads", [ctx], [act], rule=[(0, [])])[0]
        o = linear(f"{pfx}.proj", ctx, D, D)
        return dropout(f"{pfx}.resid", o, B * S * D)

    def mlp(pfx: str, h: int) -> int:
        f = linear(f"{pfx}.fc1", h, D, F)
        g = gelu(f"{pfx}.gelu", f)
        m = linear(f"{pfx}.fc2", g, F, D)
        return dropout(f"{pfx}.resid", m, B * S * D)

    if not shape.decoder:
        x = layer_norm("embed.ln", x)
    x = dropout("embed", x, B * S * D)
    for L in range(shape.layers):
        p = f"h{L}"
        if shape.decoder:   # pre-LN (GPT-2)
            a = attention(f"{p}.attn", layer_norm(f"{p}.ln1", x))
            x = b.fwd(f"{p}.add1", [x, a], [act], rule=[(0, []), (1, [])])[0]
            m = mlp(f"{p}.mlp", layer_norm(f"{p}.ln2", x))
            x = b.fwd(f"{p}.add2", [x, m], [act], rule=[(0, []), (1, [])])[0]
        else:               # post-LN (BERT)
            a = attention(f"{p}.attn", x)
            x = layer_norm(f"{p}.ln1", b.fwd(f"{p}.add1", [x, a], [act], rule=[(0, []), (1, [])])[0])
            m = mlp(f"{p}.mlp", x)
            x = layer_norm(f"{p}.ln2", b.fwd(f"{p}.add2", [x, m], [act], rule=[(0, []), (1, [])])[0])
    if shape.decoder:
        x = layer_norm("ln_f", x)
    else:  # MLM transform head
        x = linear("mlm.dense", x, D, D)
        x = b.fwd("mlm.act", [x], [act], rule=[(0, [0])])[0]
        x = layer_norm("mlm.ln", x)
    logits = b.fwd("lm_head.mm", [x], [B * S * V * f4], rule=[(("W", V * D * f4), [0]), (0, [])])[0]
    lsm = b.fwd("loss.log_softmax", [logits], [B * S * V * f4], rule=[(0, [OUT(0)])])[0]
    b.fwd("loss.nll", [lsm, labels], [f4], rule=[(0, [1])], kind="loss")
    # the loss op emits the seed gradient d(loss)/d(log_softmax) ...
    b.backward(lsm, B * S * V * f4)
    b.adam(shape.traced)
    return b.doc()


def doc_sha256(doc: dict) -> str:
    return hashlib.sha256(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def config_doc(name: str) -> dict:
    """Interchange document of a BASELINE.json config graph by name."""
    if name == "layered":
        return layered_dag_doc()
    if name in SHAPES:
        return transformer_training_doc(SHAPES[name])
    raise ValueError(f"unknown config graph {name!r}")
