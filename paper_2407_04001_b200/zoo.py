"""Seeded / deterministic INPUT generators: computation graphs G=(V,E).

This module is shared by the product path and by the oracle tests, so it holds
NONE of the method's arithmetic: no configuration enumeration, no cost model,
no ordering, no DP.  It only emits graphs in the JSON-able schema of
DESIGN.md §3 (an extension of SPEC.md:97 "JSON graph schema"):

    node = {"id", "name", "kind",
            "dims": [{"name", "size", "splittable"}],      # iteration space (§2)
            "out_axes": [iter-dim index per output-tensor axis],
            "w_axes":   [iter-dim index per weight axis]   ([] = no weight),
            "flop_dims": null | [iter-dim indices]          (null = all dims),
            "flops_per_point": int,                         (fwd+bwd FLOPs per iteration point)
            "halo": [[spatial_dim, filter_dim], ...],       (conv halo pairs)
            "in_axes":  [iter-dim index per input-tensor axis] ([] = not given; required with a
                                                             halo: the halo face, DESIGN reading L)
            "elem_bytes": int}
    edge = {"src", "dst", "axis_map": [dst iter-dim per src output axis, -1 = none]}
    graph = {"nodes": [...], "edges": [...], "machine": {"flops": F, "bandwidth": B}}

The five benchmark graphs follow SURVEY.md §8.d.1 (shapes of the paper's
networks; Table 2 dimension letters PAPER.md:923-975).
Per-kind conventions are SURVEY.md §8.b "Per-kind defaults in the zoo".
"""
from __future__ import annotations

import random
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

DEFAULT_MACHINE = {"flops": 1.0e13, "bandwidth": 1.0e10}  # r = F/B = 1000 (reading R)


class GraphBuilder:
    """Accumulates nodes/edges; dims and edge maps are given by dim NAME."""

    def __init__(self) -> None:
        self.nodes: List[dict] = []
        self.edges: List[dict] = []

    def node(self, name: str, kind: str, dims: Sequence[Tuple], out: Sequence[str],
             w: Sequence[str] = (), fpp: int = 2, flop_dims: Optional[Sequence[str]] = None,
             halo: Sequence[Tuple[str, str]] = (), elem_bytes: int = 4,
             unsplittable: Iterable[str] = (), inp: Sequence[str] = ()) -> int:
        names = [d[0] for d in dims]
        assert len(set(names)) == len(names), f"duplicate dim names in {name}"
        nosplit = set(unsplittable)
        dd = []
        for d in dims:
            split = d[2] if len(d) > 2 else (d[0] not in nosplit)
            dd.append({"name": d[0], "size": int(d[1]), "splittable": bool(split)})
        idx = {n: i for i, n in enumerate(names)}
        nid = len(self.nodes)
        self.nodes.append({
            "id": nid, "name": name, "kind": kind, "dims": dd,
            "out_axes": [idx[a] for a in out],
            "w_axes": [idx[a] for a in w],
            "flop_dims": None if flop_dims is None else [idx[a] for a in flop_dims],
            "flops_per_point": int(fpp),
            "halo": [[idx[h], idx[r]] for h, r in halo],
            "elem_bytes": int(elem_bytes),
            "in_axes": [idx[a] for a in inp],
        })
        return nid

    def edge(self, src: int, dst: int, rename: Optional[Dict[str, Optional[str]]] = None) -> None:
        """Tensor flowing src -> dst; each src output axis maps to the dst dim of
        the same name (or ``rename[name]``); absent / None means -1 (unsplit)."""
        rename = rename or {}
        s, d = self.nodes[src], self.nodes[dst]
        dnames = {x["name"]: i for i, x in enumerate(d["dims"])}
        amap = []
        for a in s["out_axes"]:
            an = s["dims"][a]["name"]
            tgt = rename.get(an, an)
            amap.append(dnames[tgt] if tgt is not None and tgt in dnames else -1)
        self.edges.append({"src": src, "dst": dst, "axis_map": amap})

    def graph(self, machine: Optional[dict] = None) -> dict:
        return {"nodes": self.nodes, "edges": self.edges,
                "machine": dict(machine or DEFAULT_MACHINE)}


# ----------------------------------------------------------------------------
# Config 1: 4-layer MLP (BASELINE.json configs[0]); SURVEY.md §8.d.1 row 1
# ----------------------------------------------------------------------------
def mlp(layers: int = 4, batch: int = 64, hidden: int = 256) -> dict:
    g = GraphBuilder()
    prev = None
    for l in range(layers):
        n = g.node(f"fc{l}", "gemm", [("b", batch), ("n", hidden), ("c", hidden)],
                   out=["b", "n"], w=["n", "c"], fpp=6)
        if prev is not None:
            g.edge(prev, n, {"n": "c"})
        prev = n
    return g.graph()


def gemm_single(m: int = 1024, n: int = 1024, k: int = 1024) -> dict:
    """Single GEMM vertex (SPEC.md:198 closed form: 6*M*N*K at the all-ones config)."""
    g = GraphBuilder()
    g.node("gemm", "gemm", [("b", m), ("n", n), ("c", k)], out=["b", "n"], w=["n", "c"], fpp=6)
    return g.graph()


# ----------------------------------------------------------------------------
# Config 2: AlexNet, batch 128 (PAPER.md:716-718 path graph; Table 2 bchwnrs/bnc/bn)
# ----------------------------------------------------------------------------
def _conv(g: GraphBuilder, name: str, b: int, cin: int, h: int, w: int, cout: int,
          r: int, s: int) -> int:
    return g.node(name, "conv2d",
                  [("b", b), ("c", cin), ("h", h), ("w", w), ("n", cout), ("r", r), ("s", s)],
                  out=["b", "n", "h", "w"], w=["c", "n", "r", "s"], fpp=6,
                  halo=[("h", "r"), ("w", "s")], unsplittable=("r", "s"), inp=["b", "c", "h", "w"])


def _pool(g: GraphBuilder, name: str, b: int, c: int, h: int, w: int, r: int, s: int) -> int:
    return g.node(name, "pool", [("b", b), ("c", c), ("h", h), ("w", w), ("r", r), ("s", s)],
                  out=["b", "c", "h", "w"], fpp=2, unsplittable=("r", "s"))


def _fc(g: GraphBuilder, name: str, b: int, n: int, c: int) -> int:
    return g.node(name, "gemm", [("b", b), ("n", n), ("c", c)], out=["b", "n"], w=["n", "c"], fpp=6)


def alexnet(batch: int = 128) -> dict:
    g = GraphBuilder()
    b = batch
    seq = [
        _conv(g, "conv1", b, 3, 55, 55, 96, 11, 11),
        _pool(g, "pool1", b, 96, 27, 27, 3, 3),
        _conv(g, "conv2", b, 96, 27, 27, 256, 5, 5),
        _pool(g, "pool2", b, 256, 13, 13, 3, 3),
        _conv(g, "conv3", b, 256, 13, 13, 384, 3, 3),
        _conv(g, "conv4", b, 384, 13, 13, 384, 3, 3),
        _conv(g, "conv5", b, 384, 13, 13, 256, 3, 3),
        _pool(g, "pool3", b, 256, 6, 6, 3, 3),
        _fc(g, "fc1", b, 4096, 9216),
        _fc(g, "fc2", b, 4096, 4096),
        _fc(g, "fc3", b, 1000, 4096),
        g.node("softmax", "softmax", [("b", b), ("n", 1000)], out=["b", "n"], fpp=10),
    ]
    kinds = [g.nodes[i]["kind"] for i in seq]
    for a, c in zip(seq, seq[1:]):
        ka, kc = g.nodes[a]["kind"], g.nodes[c]["kind"]
        if ka == "conv2d":                    # conv out (b,n,h,w) -> next in-channel c
            g.edge(a, c, {"n": "c"})
        elif ka == "pool" and kc == "gemm":   # flatten (b,c,h,w) -> fc (b,n,c): c->c, h,w folded
            g.edge(a, c, {"h": None, "w": None})
        elif ka == "gemm":                    # fc out (b,n) -> next in-dim c (or softmax n)
            g.edge(a, c, {"n": "c"} if kc == "gemm" else None)
        else:
            g.edge(a, c)
    del kinds
    return g.graph()


# ----------------------------------------------------------------------------
# Config 3: InceptionV3, batch 128, 218 vertices (SURVEY.md §8.c.3 reconstruction)
# PAPER.md:680-683 "218 nodes, of which 206 ... degree < 5 and ... 12 ... >= 5";
# PAPER.md:703-704 "Nodes 171 and 193 have high degree" (InceptionE module).
# ----------------------------------------------------------------------------
class _Inception:
    def __init__(self, batch: int):
        self.g = GraphBuilder()
        self.b = batch

    def conv_bn(self, name: str, src: Optional[int], cin: int, hin: int, win: int,
                cout: int, r: int, s: int, stride: int = 1, pad: bool = True) -> Tuple[int, int, int]:
        """conv vertex + BN/ReLU vertex; returns (bn id, h_out, w_out)."""
        if pad and stride == 1:
            ho, wo = hin, win
        else:
            ho, wo = (hin - r) // stride + 1, (win - s) // stride + 1
        g = self.g
        cv = _conv(g, name, self.b, cin, ho, wo, cout, r, s)
        if src is not None:
            g.edge(src, cv, {"n": "c"} if g.nodes[src]["kind"] == "conv2d" else None)
        bn = g.node(name + "/bn", "bn_relu", [("b", self.b), ("c", cout), ("h", ho), ("w", wo)],
                    out=["b", "c", "h", "w"], w=["c"], fpp=10)
        g.edge(cv, bn, {"n": "c"})
        return bn, ho, wo

    def pool(self, name: str, src: int, c: int, hin: int, win: int, k: int, stride: int,
             pad: bool) -> Tuple[int, int, int]:
        if pad and stride == 1:
            ho, wo = hin, win
        else:
            ho, wo = (hin - k) // stride + 1, (win - k) // stride + 1
        p = _pool(self.g, name, self.b, c, ho, wo, k, k)
        self.g.edge(src, p)
        return p, ho, wo

    def concat(self, name: str, srcs: Sequence[int], ctot: int, h: int, w: int) -> int:
        g = self.g
        cc = g.node(name, "concat", [("b", self.b), ("c", ctot), ("h", h), ("w", w)],
                    out=["b", "c", "h", "w"], fpp=2)
        for s_ in srcs:
            g.edge(s_, cc)
        return cc


def inception_v3(batch: int = 128) -> dict:
    I = _Inception(batch)
    # Stem (12 vertices): 5 conv+bn pairs + 2 max-pools; 299x299x3 input.
    x, h, w = I.conv_bn("Conv2d_1a_3x3", None, 3, 299, 299, 32, 3, 3, stride=2, pad=False)
    x, h, w = I.conv_bn("Conv2d_2a_3x3", x, 32, h, w, 32, 3, 3, pad=False, stride=1)
    x, h, w = I.conv_bn("Conv2d_2b_3x3", x, 32, h, w, 64, 3, 3)
    x, h, w = I.pool("MaxPool_3a_3x3", x, 64, h, w, 3, 2, pad=False)
    x, h, w = I.conv_bn("Conv2d_3b_1x1", x, 64, h, w, 80, 1, 1)
    x, h, w = I.conv_bn("Conv2d_4a_3x3", x, 80, h, w, 192, 3, 3, pad=False, stride=1)
    x, h, w = I.pool("MaxPool_5a_3x3", x, 192, h, w, 3, 2, pad=False)
    c = 192
    # 3 x InceptionA (16 vertices each)
    for name, pool_c in (("Mixed_5b", 32), ("Mixed_5c", 64), ("Mixed_5d", 64)):
        b0, _, _ = I.conv_bn(name + "/b0_1x1", x, c, h, w, 64, 1, 1)
        b1, _, _ = I.conv_bn(name + "/b1_1x1", x, c, h, w, 48, 1, 1)
        b1, _, _ = I.conv_bn(name + "/b1_5x5", b1, 48, h, w, 64, 5, 5)
        b2, _, _ = I.conv_bn(name + "/b2_1x1", x, c, h, w, 64, 1, 1)
        b2, _, _ = I.conv_bn(name + "/b2_3x3a", b2, 64, h, w, 96, 3, 3)
        b2, _, _ = I.conv_bn(name + "/b2_3x3b", b2, 96, h, w, 96, 3, 3)
        b3, _, _ = I.pool(name + "/b3_avgpool", x, c, h, w, 3, 1, pad=True)
        b3, _, _ = I.conv_bn(name + "/b3_1x1", b3, c, h, w, pool_c, 1, 1)
        c = 64 + 64 + 96 + pool_c
        x = I.concat(name + "/concat", [b0, b1, b2, b3], c, h, w)
    # InceptionB (Mixed_6a, 10 vertices)
    b0, h2, w2 = I.conv_bn("Mixed_6a/b0_3x3", x, c, h, w, 384, 3, 3, stride=2, pad=False)
    b1, _, _ = I.conv_bn("Mixed_6a/b1_1x1", x, c, h, w, 64, 1, 1)
    b1, _, _ = I.conv_bn("Mixed_6a/b1_3x3a", b1, 64, h, w, 96, 3, 3)
    b1, _, _ = I.conv_bn("Mixed_6a/b1_3x3b", b1, 96, h, w, 96, 3, 3, stride=2, pad=False)
    b2, _, _ = I.pool("Mixed_6a/b2_maxpool", x, c, h, w, 3, 2, pad=False)
    h, w = h2, w2
    c = 384 + 96 + c
    x = I.concat("Mixed_6a/concat", [b0, b1, b2], c, h, w)
    # 4 x InceptionC (22 vertices each)
    for name, c7 in (("Mixed_6b", 128), ("Mixed_6c", 160), ("Mixed_6d", 160), ("Mixed_6e", 192)):
        b0, _, _ = I.conv_bn(name + "/b0_1x1", x, c, h, w, 192, 1, 1)
        b1, _, _ = I.conv_bn(name + "/b1_1x1", x, c, h, w, c7, 1, 1)
        b1, _, _ = I.conv_bn(name + "/b1_1x7", b1, c7, h, w, c7, 1, 7)
        b1, _, _ = I.conv_bn(name + "/b1_7x1", b1, c7, h, w, 192, 7, 1)
        b2, _, _ = I.conv_bn(name + "/b2_1x1", x, c, h, w, c7, 1, 1)
        b2, _, _ = I.conv_bn(name + "/b2_7x1a", b2, c7, h, w, c7, 7, 1)
        b2, _, _ = I.conv_bn(name + "/b2_1x7a", b2, c7, h, w, c7, 1, 7)
        b2, _, _ = I.conv_bn(name + "/b2_7x1b", b2, c7, h, w, c7, 7, 1)
        b2, _, _ = I.conv_bn(name + "/b2_1x7b", b2, c7, h, w, 192, 1, 7)
        b3, _, _ = I.pool(name + "/b3_avgpool", x, c, h, w, 3, 1, pad=True)
        b3, _, _ = I.conv_bn(name + "/b3_1x1", b3, c, h, w, 192, 1, 1)
        c = 768
        x = I.concat(name + "/concat", [b0, b1, b2, b3], c, h, w)
    # InceptionD (Mixed_7a, 14 vertices) -> concat is vertex 171
    b0, _, _ = I.conv_bn("Mixed_7a/b0_1x1", x, c, h, w, 192, 1, 1)
    b0, h2, w2 = I.conv_bn("Mixed_7a/b0_3x3", b0, 192, h, w, 320, 3, 3, stride=2, pad=False)
    b1, _, _ = I.conv_bn("Mixed_7a/b1_1x1", x, c, h, w, 192, 1, 1)
    b1, _, _ = I.conv_bn("Mixed_7a/b1_1x7", b1, 192, h, w, 192, 1, 7)
    b1, _, _ = I.conv_bn("Mixed_7a/b1_7x1", b1, 192, h, w, 192, 7, 1)
    b1, _, _ = I.conv_bn("Mixed_7a/b1_3x3", b1, 192, h, w, 192, 3, 3, stride=2, pad=False)
    b2, _, _ = I.pool("Mixed_7a/b2_maxpool", x, c, h, w, 3, 2, pad=False)
    h, w = h2, w2
    c = 320 + 192 + c
    x = I.concat("Mixed_7a/concat", [b0, b1, b2], c, h, w)
    # 2 x InceptionE (22 vertices each) -> concats 193, 215
    for name in ("Mixed_7b", "Mixed_7c"):
        b0, _, _ = I.conv_bn(name + "/b0_1x1", x, c, h, w, 320, 1, 1)
        b1, _, _ = I.conv_bn(name + "/b1_1x1", x, c, h, w, 384, 1, 1)
        b1a, _, _ = I.conv_bn(name + "/b1_1x3", b1, 384, h, w, 384, 1, 3)
        b1b, _, _ = I.conv_bn(name + "/b1_3x1", b1, 384, h, w, 384, 3, 1)
        b1 = I.concat(name + "/b1_concat", [b1a, b1b], 768, h, w)
        b2, _, _ = I.conv_bn(name + "/b2_1x1", x, c, h, w, 448, 1, 1)
        b2, _, _ = I.conv_bn(name + "/b2_3x3", b2, 448, h, w, 384, 3, 3)
        b2a, _, _ = I.conv_bn(name + "/b2_1x3", b2, 384, h, w, 384, 1, 3)
        b2b, _, _ = I.conv_bn(name + "/b2_3x1", b2, 384, h, w, 384, 3, 1)
        b2 = I.concat(name + "/b2_concat", [b2a, b2b], 768, h, w)
        b3, _, _ = I.pool(name + "/b3_avgpool", x, c, h, w, 3, 1, pad=True)
        b3, _, _ = I.conv_bn(name + "/b3_1x1", b3, c, h, w, 192, 1, 1)
        c = 320 + 768 + 768 + 192
        x = I.concat(name + "/concat", [b0, b1, b2, b3], c, h, w)
    # Head (2 vertices): FC (global pool folded: h,w -> unsplit) + softmax.
    g = I.g
    fc = _fc(g, "Logits/fc", batch, 1000, c)
    g.edge(x, fc, {"h": None, "w": None})
    sm = g.node("Predictions/softmax", "softmax", [("b", batch), ("n", 1000)], out=["b", "n"], fpp=10)
    g.edge(fc, sm)
    return g.graph()


# ----------------------------------------------------------------------------
# Config 4: unrolled RNNLM / GNMT (FlexFlow-style unroll 40)
# ----------------------------------------------------------------------------
def _lstm_cell(g: GraphBuilder, name: str, b: int, hidden: int, din: int) -> int:
    # one GEMM over [x; h]: gates n = 4*hidden, reduction c = din + hidden
    return g.node(name, "lstm_cell", [("b", b), ("n", 4 * hidden), ("c", din + hidden)],
                  out=["b", "n"], w=["n", "c"], fpp=6)


def _embedding(g: GraphBuilder, name: str, b: int, d: int, v: int) -> int:
    return g.node(name, "embedding", [("b", b), ("d", d), ("v", v)], out=["b", "d"],
                  w=["d", "v"], fpp=2, flop_dims=["b", "d"])


def _proj(g: GraphBuilder, name: str, b: int, v: int, d: int) -> int:
    return g.node(name, "gemm", [("b", b), ("v", v), ("d", d)], out=["b", "v"], w=["v", "d"], fpp=6)


def rnnlm_unrolled(layers: int = 2, steps: int = 40, batch: int = 64, hidden: int = 1024,
                   vocab: int = 32768) -> dict:
    """Ladder grid: emb(t) -> cell(0,t) -> ... -> cell(L-1,t) -> proj(t) -> softmax(t);
    cell(l,t) -> cell(l,t+1) carries the recurrent state."""
    g = GraphBuilder()
    cell = {}
    for t in range(steps):
        e = _embedding(g, f"emb{t}", batch, hidden, vocab)
        prev = e
        for l in range(layers):
            c = _lstm_cell(g, f"lstm{l}_{t}", batch, hidden, hidden)
            cell[l, t] = c
            g.edge(prev, c, {"d": "c", "n": "c"})
            if t > 0:
                g.edge(cell[l, t - 1], c, {"n": "c"})
            prev = c
        pj = _proj(g, f"proj{t}", batch, vocab, hidden)
        g.edge(prev, pj, {"n": "d"})
        sm = g.node(f"softmax{t}", "softmax", [("b", batch), ("v", vocab)], out=["b", "v"], fpp=10)
        g.edge(pj, sm)
    return g.graph()


def gnmt_unrolled(layers: int = 2, steps: int = 40, batch: int = 64, hidden: int = 1024,
                  vocab: int = 32768) -> dict:
    """Encoder ladder (layers x steps) -> encoder memory node; decoder ladder with
    per-step attention over the memory and input feeding attn(t) -> dec cell(0,t+1)."""
    g = GraphBuilder()
    enc = {}
    for t in range(steps):
        prev = _embedding(g, f"enc_emb{t}", batch, hidden, vocab)
        for l in range(layers):
            c = _lstm_cell(g, f"enc{l}_{t}", batch, hidden, hidden)
            enc[l, t] = c
            g.edge(prev, c, {"d": "c", "n": "c"})
            if t > 0:
                g.edge(enc[l, t - 1], c, {"n": "c"})
            prev = c
    # memory: all top-layer encoder outputs, (b, s, e)
    mem = g.node("enc_memory", "concat", [("b", batch), ("s", steps), ("e", 4 * hidden)],
                 out=["b", "s", "e"], fpp=2)
    for t in range(steps):
        g.edge(enc[layers - 1, t], mem, {"n": "e"})
    dec = {}
    attn_prev = None
    for t in range(steps):
        prev = _embedding(g, f"dec_emb{t}", batch, hidden, vocab)
        for l in range(layers):
            c = _lstm_cell(g, f"dec{l}_{t}", batch, hidden, hidden)
            dec[l, t] = c
            g.edge(prev, c, {"d": "c", "n": "c"})
            if t > 0:
                g.edge(dec[l, t - 1], c, {"n": "c"})
            if l == 0 and attn_prev is not None:
                g.edge(attn_prev, c, {"e": "c"})           # input feeding
            prev = c
        at = g.node(f"attn{t}", "attention", [("b", batch), ("s", steps), ("e", 4 * hidden)],
                    out=["b", "e"], fpp=6)
        g.edge(mem, at)
        g.edge(prev, at, {"n": "e"})
        attn_prev = at
        pj = _proj(g, f"proj{t}", batch, vocab, 4 * hidden)
        g.edge(at, pj, {"e": "d"})
        sm = g.node(f"softmax{t}", "softmax", [("b", batch), ("v", vocab)], out=["b", "v"], fpp=10)
        g.edge(pj, sm)
    return g.graph()


# ----------------------------------------------------------------------------
# Config 5: Transformer 6+6, d_model 1024 (Table 2 bshck/bsde/bsvd)
# ----------------------------------------------------------------------------
def transformer(enc_layers: int = 6, dec_layers: int = 6, batch: int = 64, seq: int = 256,
                d_model: int = 1024, heads: int = 16, d_ff: int = 4096, vocab: int = 32768) -> dict:
    g = GraphBuilder()
    b, s, d, h, e, v = batch, seq, d_model, heads, d_ff, vocab
    c = d_model // heads

    def proj(name):      # q/k/v projection (b,s,h,c,d)
        return g.node(name, "qkv_proj", [("b", b), ("s", s), ("h", h), ("c", c), ("d", d)],
                      out=["b", "s", "h", "c"], w=["h", "c", "d"], fpp=6)

    def layernorm(name):
        return g.node(name, "add_layernorm", [("b", b), ("s", s), ("d", d)],
                      out=["b", "s", "d"], w=["d"], fpp=10)

    def attention(pfx: str, xq: int, xkv: int) -> int:
        q, k, vv = proj(pfx + "/q"), proj(pfx + "/k"), proj(pfx + "/v")
        g.edge(xq, q)
        g.edge(xkv, k)
        g.edge(xkv, vv)
        sc = g.node(pfx + "/score", "attn_score", [("b", b), ("h", h), ("sq", s), ("sk", s), ("c", c)],
                    out=["b", "h", "sq", "sk"], fpp=6)
        g.edge(q, sc, {"s": "sq"})
        g.edge(k, sc, {"s": "sk"})
        sm = g.node(pfx + "/softmax", "softmax", [("b", b), ("h", h), ("sq", s), ("sk", s)],
                    out=["b", "h", "sq", "sk"], fpp=10)
        g.edge(sc, sm)
        cx = g.node(pfx + "/context", "attn_context", [("b", b), ("h", h), ("sq", s), ("c", c), ("sk", s)],
                    out=["b", "h", "sq", "c"], fpp=6)
        g.edge(sm, cx)
        g.edge(vv, cx, {"s": "sk"})
        op = g.node(pfx + "/out_proj", "out_proj", [("b", b), ("s", s), ("d", d), ("h", h), ("c", c)],
                    out=["b", "s", "d"], w=["d", "h", "c"], fpp=6)
        g.edge(cx, op, {"sq": "s"})
        ln = layernorm(pfx + "/add_ln")
        g.edge(op, ln)
        g.edge(xq, ln)                                   # residual
        return ln

    def ffn(pfx: str, x: int) -> int:
        f1 = g.node(pfx + "/ff1", "gemm", [("b", b), ("s", s), ("e", e), ("d", d)],
                    out=["b", "s", "e"], w=["e", "d"], fpp=6)
        g.edge(x, f1)
        f2 = g.node(pfx + "/ff2", "gemm", [("b", b), ("s", s), ("d", d), ("e", e)],
                    out=["b", "s", "d"], w=["d", "e"], fpp=6)
        g.edge(f1, f2)
        ln = layernorm(pfx + "/add_ln_ff")
        g.edge(f2, ln)
        g.edge(x, ln)
        return ln

    def embedding(name):
        return g.node(name, "embedding", [("b", b), ("s", s), ("d", d), ("v", v)],
                      out=["b", "s", "d"], w=["d", "v"], fpp=2, flop_dims=["b", "s", "d"])

    x = embedding("enc_embedding")
    for l in range(enc_layers):
        x = attention(f"enc{l}/self_attn", x, x)
        x = ffn(f"enc{l}", x)
    enc_out = x                                           # long live range
    y = embedding("dec_embedding")
    for l in range(dec_layers):
        y = attention(f"dec{l}/self_attn", y, y)
        y = attention(f"dec{l}/cross_attn", y, enc_out)
        y = ffn(f"dec{l}", y)
    fp = g.node("final_proj", "gemm", [("b", b), ("s", s), ("v", v), ("d", d)],
                out=["b", "s", "v"], w=["v", "d"], fpp=6)
    g.edge(y, fp)
    sm = g.node("softmax", "softmax", [("b", b), ("s", s), ("v", v)], out=["b", "s", "v"], fpp=10)
    g.edge(fp, sm)
    return g.graph()


# ----------------------------------------------------------------------------
# Toy graph of Fig. 3, reconstructed:
# with sigma = (1..9) and edges {1-2, 2-5, 3-5, 5-8, 4-7, 4-9, 6-7, 7-8, 8-9, 6-9}
# X(5) = {1,2,3,5}, S(5) = {{1,2},{3}}, D(5) = {8}, Dbar(5) = {7,8,9}.
# Node id k-1 is sigma_k of the depicted ordering.
# ----------------------------------------------------------------------------
TOY_EDGES_1BASED = [(1, 2), (2, 5), (3, 5), (5, 8), (4, 7), (4, 9), (6, 7), (7, 8), (8, 9), (6, 9)]


def toy_fig3(p_dim: int = 4) -> dict:
    g = GraphBuilder()
    for k in range(1, 10):
        g.node(f"v{k}", "gemm", [("b", 8), ("n", p_dim), ("c", p_dim)], out=["b", "n"], w=["n", "c"], fpp=6)
    for a, c in TOY_EDGES_1BASED:
        g.edge(a - 1, c - 1, {"n": "c"})
    return g.graph()


# ----------------------------------------------------------------------------
# Seeded random weakly connected graphs (SURVEY.md §4 "Fixtures to build").
# ----------------------------------------------------------------------------
def random_topology(n: int, seed: int, extra_p: float = 0.3,
                    multi_p: float = 0.0) -> List[Tuple[int, int]]:
    """Random spanning tree (each vertex k>0 attaches to a random earlier vertex,
    ids then shuffled) plus extra edges with probability extra_p; random direction.
    multi_p adds parallel / antiparallel duplicates (multigraph reading M)."""
    rng = random.Random(seed)
    perm = list(range(n))
    rng.shuffle(perm)
    edges = []
    for k in range(1, n):
        a, c = perm[k], perm[rng.randrange(k)]
        edges.append((a, c) if rng.random() < 0.5 else (c, a))
    have = {frozenset(e) for e in edges}
    for a in range(n):
        for c in range(a + 1, n):
            if frozenset((a, c)) not in have and rng.random() < extra_p:
                edges.append((a, c) if rng.random() < 0.5 else (c, a))
    if multi_p > 0:
        for (a, c) in list(edges):
            if rng.random() < multi_p:
                edges.append((c, a) if rng.random() < 0.5 else (a, c))
    rng.shuffle(edges)
    return edges


def random_chain_graph(n: int, seed: int, kmax: int = 12, extra_p: float = 0.3,
                       multi_p: float = 0.0) -> Tuple[dict, int]:
    """Graph whose vertex v has a single splittable dim of size 2^(K_v - 1), so that
    under the LE_P policy with p = 2^(kmax-1) it has exactly K_v configs (1,2,4,..).
    Used with explicit random cost tables (pase override hook / oracle tables).
    Returns (graph, p)."""
    rng = random.Random(seed * 7919 + 17)
    g = GraphBuilder()
    for i in range(n):
        K = rng.randint(1, kmax)
        g.node(f"r{i}", "synthetic", [("x", 1 << (K - 1))], out=["x"], fpp=1)
    for a, c in random_topology(n, seed, extra_p, multi_p):
        g.edge(a, c, {"x": None})
    return g.graph(), 1 << (kmax - 1)


def random_model_graph(n: int, seed: int, extra_p: float = 0.3, max_log: int = 4,
                       multi_p: float = 0.0) -> dict:
    """Random graph with random 1-4-D iteration spaces (sizes 2^a, some odd /
    unsplittable), random output / weight axes, random axis maps and halos: exercises
    the cost model (t_l, t_x) on structures the zoo does not produce."""
    rng = random.Random(seed * 104729 + 3)
    rng_in = random.Random(seed * 7 + 11)          # input-tensor axes (own stream: same graphs)
    g = GraphBuilder()
    names = "abcdefgh"
    for i in range(n):
        d = rng.randint(1, 4)
        dims = []
        for k in range(d):
            sz = 1 << rng.randint(0, max_log)
            if rng.random() < 0.15:
                sz = rng.choice([3, 5, 6, 7, 12])
            dims.append((names[k], sz, rng.random() < 0.85))
        dn = [x[0] for x in dims]
        nout = rng.randint(1, d)
        out = rng.sample(dn, nout)
        w = rng.sample(dn, rng.randint(0, d)) if rng.random() < 0.6 else []
        fd = None if rng.random() < 0.7 else rng.sample(dn, rng.randint(1, d))
        halo = []
        if d >= 2 and rng.random() < 0.2:
            halo = [(dn[0], dn[1])]
        inp = rng_in.sample(dn, rng_in.randint(1, d))
        if halo and dn[0] not in inp:
            inp = [dn[0]] + inp[:d - 1]
        g.node(f"m{i}", "synthetic", dims, out=out, w=w, fpp=rng.choice([1, 2, 6, 10]),
               flop_dims=fd, halo=halo, elem_bytes=rng.choice([2, 4]), inp=inp)
    for a, c in random_topology(n, seed, extra_p, multi_p):
        src, dst = g.nodes[a], g.nodes[c]
        dnames = [x["name"] for x in dst["dims"]]
        rename = {}
        for ax in src["out_axes"]:
            nm = src["dims"][ax]["name"]
            rename[nm] = rng.choice(dnames + [None])
        g.edge(a, c, rename)
    return g.graph()


# ----------------------------------------------------------------------------
# Synthetic streaming-regime benchmark ("add a synthetic streaming
# benchmark: a chain whose child table spans D ∪ {σ}"); NOT a paper config.
# ----------------------------------------------------------------------------
def streaming_clique(extra: int = 3, batch: int = 64, seq: int = 256, heads: int = 16,
                     head_dim: int = 64, d_model: int = 1024) -> dict:
    """A clique of 2 + `extra` projection-shaped vertices (b, s, h, c, d: the Transformer's q/k/v
    shape, K = 205 at p = 64 under EXACT_P).  Vertex 0 has no splittable dim (K = 1), so SortNodes
    eliminates it first with D = all others: its table spans (sigma_1, D(1)) -- 205^(extra+1)
    entries (extra = 3: 1.77e9 entries, 14 GB) -- and vertex 1, eliminated next with
    D(1) = {2..}, reads each entry of it exactly once (one 8-B read per candidate, nothing reused):
    the streaming regime, where the DP fill is HBM-bound."""
    g = GraphBuilder()
    dims = [("b", batch), ("s", seq), ("h", heads), ("c", head_dim), ("d", d_model)]
    n = 2 + extra
    for i in range(n):
        g.node(f"x{i}", "qkv_proj", dims, out=["b", "s", "h", "c"], w=["h", "c", "d"], fpp=6,
               unsplittable=("b", "s", "h", "c", "d") if i == 0 else ())
    for a in range(n):
        for c in range(a + 1, n):
            g.edge(a, c)
    return g.graph()


BENCH_GRAPHS = {
    "mlp": (mlp, 4),
    "alexnet": (alexnet, 8),
    "inception_v3": (inception_v3, 32),
    "rnnlm": (rnnlm_unrolled, 64),
    "gnmt": (gnmt_unrolled, 64),
    # GNMT at 4 + 4 layers (sizing rule iii): M = 5, 7.2e10 candidates,
    # 2.6e9 table entries (26 GB of T + A): the paper-shaped config where tables leave L2
    "gnmt4": (lambda: gnmt_unrolled(layers=4), 64),
    # real GNMT depth (8 + 8): M = 15 > PASE_MAX_DEP -> PASE_ERR_RESOURCE (Table 1's "OOM" analogue)
    "gnmt8": (lambda: gnmt_unrolled(layers=8), 64),
    # synthetic streaming-regime benchmark (not a paper config): 14 GB child table read once
    "stream205": (streaming_clique, 64),
    "transformer": (transformer, 64),
    # latency microbenchmark (not a paper config): a 200-vertex path, |D(i)| = 1, K = 6
    "chain200": (lambda: mlp(layers=200), 4),
}


def bench_graph(name: str) -> Tuple[dict, int]:
    """(graph, p) for one of the BASELINE.json configs."""
    fn, p = BENCH_GRAPHS[name]
    return fn(), p
