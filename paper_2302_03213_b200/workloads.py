"""The callers either side of the LUT path, built for BASELINE.json's configs.

Synthetic, seeded, device-resident instances (there are no checkpoints or
datasets here) of:

  configs[0]/[4]  single LUT Linear               `linear`
  configs[1]      BERT-base FFN pair, int8 + GELU  `FfnPair` / `ffn_pair`
  configs[2]      ResNet20-style 3x3 LUT convs     `resnet_convs`
  configs[3]      12-layer BERT-base encoder       `BertEncoder` / `bert_encoder`

Layers are this package's LutLinear / LutConv2d, so every replaced GEMM runs
encode -> lookup-aggregate -> bias/activation epilogue in the sm_100a kernels;
attention score/softmax matmuls, LayerNorm and the dense layers a config keeps
run in torch (fp32, TF32 off).  Centroids follow SURVEY §8(d): K sub-vectors
sampled from a held-out calibration batch of the layer's own input
distribution (the rule `init_from_float` approximates with k-means,
model.py:314-359); tables are built from the dense weights by the table
kernels (pq.py:177-193, quant.py:40-57).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .errors import ConfigError
from .layer import LutLayer
from .nn import LutConv2d, LutLinear
from .pq import PqConfig


def _gen(dev, seed):
    return torch.Generator(device=dev).manual_seed(seed)


def sample_centroids(held: torch.Tensor, v: int, k: int, gen: torch.Generator) -> torch.Tensor:
    """(C, K, V) books: for each codebook, the sub-vectors of K distinct random
    rows of the held-out batch `held` (N, C*V)."""
    n, d = held.shape
    if d % v:
        raise ConfigError(f"D={d} not divisible by V={v}")
    if n < k:
        raise ConfigError(f"held-out batch has {n} rows < K={k}")
    c = d // v
    rows = torch.stack([torch.randperm(n, generator=gen, device=held.device)[:k] for _ in range(c)])  # (C, K)
    sub = held.reshape(n, c, v)
    return sub[rows, torch.arange(c, device=held.device)[:, None]].contiguous()


def lut_from_dense(weight_dm: torch.Tensor, bias, held: torch.Tensor, v: int, k: int, gen, integer=True,
                   act=None, scale_mtile: int = 0, gather: str = "auto", per_codebook: bool = False) -> LutLayer:
    """Replace a (D, M) weight by a LUT layer whose centroids come from `held`."""
    books = sample_centroids(held, v, k, gen)
    return LutLayer(cfg=PqConfig(v=v, k=k), books=books, weight=weight_dm, bias=bias, qat=integer, act=act,
                    scale_mtile=scale_mtile, device=weight_dm.device, gather=gather, scale_per_codebook=per_codebook)


def standardize(x: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    """LayerNorm-like standardisation over the last dim (configs[1] inputs)."""
    return (x - x.mean(-1, keepdim=True)) / torch.sqrt(x.var(-1, unbiased=False, keepdim=True) + eps)


# ----------------------------------------------------------------- configs[0]/[4]


def linear(dev, rows: int, d: int, m: int, v: int, k: int, integer: bool, seed: int = 1234,
           gather: str = "auto", scale: float | None = None):
    """Single LUT Linear: A, books ~N(0,1); W ~N(0, 1/D) (or `scale`); zero bias."""
    g = _gen(dev, seed)
    books = torch.randn((d // v, k, v), generator=g, device=dev)
    w = torch.randn((d, m), generator=g, device=dev) * (scale if scale is not None else 1.0 / math.sqrt(d))
    layer = LutLayer(cfg=PqConfig(v=v, k=k), books=books, weight=w, qat=integer, device=dev, gather=gather)
    a = torch.randn((rows, d), generator=_gen(dev, seed + 1), device=dev)
    return layer, a


# ------------------------------------------------------------------- configs[1]


class FfnPair(torch.nn.Module):
    """768 -> 3072 (GELU fused in the gather epilogue) -> 768, int8 tables."""

    def __init__(self, up: LutLayer, down: LutLayer):
        super().__init__()
        self.up = LutLinear(up)
        self.down = LutLinear(down)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return self.down(self.up(x))


def ffn_pair(dev, tokens: int = 4096, hidden: int = 768, ffn: int = 3072, v: int = 32, k: int = 16,
             scale_mtile: int = 0, seed: int = 2024, held_rows: int = 4096, gather: str = "auto",
             per_codebook: bool = False):
    """configs[1]: inputs standardised N(0,1); W ~N(0, 0.02); centroids from a
    held-out batch (FFN2's from GELU(FFN1) of that batch, dense); int8 tables,
    one scale per table (parity), per m-tile (`scale_mtile`) or per (codebook,
    m-tile) (`per_codebook`, BASELINE's wording; extensions)."""
    g = _gen(dev, seed)
    w1 = torch.randn((hidden, ffn), generator=g, device=dev) * 0.02
    w2 = torch.randn((ffn, hidden), generator=g, device=dev) * 0.02
    held = standardize(torch.randn((held_rows, hidden), generator=g, device=dev))
    up = lut_from_dense(w1, None, held, v, k, g, act="gelu", scale_mtile=scale_mtile, gather=gather,
                        per_codebook=per_codebook)
    held2 = F.gelu(_mm(held, w1))
    down = lut_from_dense(w2, None, held2, v, k, g, scale_mtile=scale_mtile, gather=gather,
                          per_codebook=per_codebook)
    x = standardize(torch.randn((tokens, hidden), generator=_gen(dev, seed + 1), device=dev))
    return FfnPair(up, down), x


def _mm(a, b):
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return a @ b
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


# ------------------------------------------------------------------- configs[2]


RESNET_STAGES = ((16, 32), (32, 16), (64, 8))  # (channels, spatial)


def resnet_convs(dev, batch: int = 256, k: int = 16, seed: int = 2020, stages=RESNET_STAGES,
                 held_batch: int = 8):
    """configs[2]: one 3x3/s1/p1 LUT conv per stage, V=9 (one input channel's
    patch), C=Cin, Cout=Cin, W ~N(0, 2/(9 Cin)), fp32 tables; inputs are
    post-ReLU |N(0,1)| NCHW; centroids from im2col patches of a held-out batch."""
    from .tensor import im2col

    out = []
    for i, (ch, hw) in enumerate(stages):
        g = _gen(dev, seed + 17 * i)
        w = torch.randn((ch * 9, ch), generator=g, device=dev) * math.sqrt(2.0 / (9 * ch))
        held = torch.randn((held_batch, ch, hw, hw), generator=g, device=dev).abs()
        lut = lut_from_dense(w, None, im2col(held, 3, 3, 1, 1), 9, k, g, integer=False)
        x = torch.randn((batch, ch, hw, hw), generator=_gen(dev, seed + 17 * i + 1), device=dev).abs()
        out.append((LutConv2d(ch, 3, 1, 1, lut), x))
    return out


# ------------------------------------------------------------------- configs[3]


@dataclass(frozen=True)
class BertConfig:
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    layers: int = 12
    dense_layers: int = 2     # layers 1-2 kept dense
    v: int = 32
    k: int = 16
    ln_eps: float = 1e-12


class _Dense(torch.nn.Module):
    def __init__(self, w_dm: torch.Tensor, b: torch.Tensor, act=None):
        super().__init__()
        self.w, self.b, self.act = w_dm, b, act

    def forward(self, x):
        y = _mm(x.reshape(-1, x.shape[-1]), self.w).reshape(*x.shape[:-1], -1) + self.b
        return F.gelu(y) if self.act == "gelu" else y


class BertLayer(torch.nn.Module):
    """Post-LN BERT block; `proj` holds q, k, v, o, up (GELU), down."""

    NAMES = ("q", "k", "v", "o", "up", "down")

    def __init__(self, cfg: BertConfig, proj: dict, ln: tuple):
        super().__init__()
        self.cfg = cfg
        self.proj = torch.nn.ModuleDict(proj)
        self.ln1_w, self.ln1_b, self.ln2_w, self.ln2_b = ln

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        b, s, h = x.shape
        nh = self.cfg.heads
        q = self.proj["q"](x).reshape(b, s, nh, h // nh).transpose(1, 2)
        k = self.proj["k"](x).reshape(b, s, nh, h // nh).transpose(1, 2)
        v = self.proj["v"](x).reshape(b, s, nh, h // nh).transpose(1, 2)
        ctx = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(b, s, h)
        x = F.layer_norm(x + self.proj["o"](ctx), (h,), self.ln1_w, self.ln1_b, self.cfg.ln_eps)
        y = self.proj["down"](self.proj["up"](x))
        return F.layer_norm(x + y, (h,), self.ln2_w, self.ln2_b, self.cfg.ln_eps)


class BertEncoder(torch.nn.Module):
    def __init__(self, cfg: BertConfig, layers: list):
        super().__init__()
        self.cfg = cfg
        self.layers = torch.nn.ModuleList(layers)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        for layer in self.layers:
            x = layer(x)
        return x

    def lut_linears(self):
        return [(i, n, layer.proj[n]) for i, layer in enumerate(self.layers) for n in BertLayer.NAMES
                if isinstance(layer.proj[n], LutLinear)]


def bert_encoder(dev, batch: int = 64, seq: int = 128, cfg: BertConfig = BertConfig(), seed: int = 4242,
                 calib_batch: int = 8, scale_mtile: int = 0, gather: str = "auto"):
    """configs[3]: random-init BERT-base (W ~N(0, 0.02), zero biases, LN = 1/0),
    random N(0,1) token embeddings; layers > `dense_layers` have every linear
    replaced by an int8 LUT layer whose centroids are sampled from that
    linear's inputs on a calibration batch run through the dense model."""
    g = _gen(dev, seed)
    h, f = cfg.hidden, cfg.ffn
    dense = []
    for _ in range(cfg.layers):
        shapes = {"q": (h, h), "k": (h, h), "v": (h, h), "o": (h, h), "up": (h, f), "down": (f, h)}
        ws = {n: torch.randn(s, generator=g, device=dev) * 0.02 for n, s in shapes.items()}
        bs = {n: torch.zeros(s[1], device=dev) for n, s in shapes.items()}
        ln = (torch.ones(h, device=dev), torch.zeros(h, device=dev), torch.ones(h, device=dev),
              torch.zeros(h, device=dev))
        dense.append((ws, bs, ln))

    # calibration pass through the dense model, capturing every linear's input
    calib = torch.randn((calib_batch, seq, h), generator=g, device=dev)
    captured: dict = {}
    x = calib
    for li, (ws, bs, ln) in enumerate(dense):
        proj = {n: _Dense(ws[n], bs[n], "gelu" if n == "up" else None) for n in BertLayer.NAMES}
        for n, mod in proj.items():
            mod.register_forward_hook(lambda m_, inp, out_, key=(li, n): captured.__setitem__(
                key, inp[0].reshape(-1, inp[0].shape[-1]).detach()))
        x = BertLayer(cfg, proj, ln)(x)

    layers = []
    for li, (ws, bs, ln) in enumerate(dense):
        if li < cfg.dense_layers:
            proj = {n: _Dense(ws[n], bs[n], "gelu" if n == "up" else None) for n in BertLayer.NAMES}
        else:
            proj = {n: LutLinear(lut_from_dense(ws[n], bs[n], captured[(li, n)], cfg.v, cfg.k, g,
                                                act="gelu" if n == "up" else None, scale_mtile=scale_mtile,
                                                gather=gather))
                    for n in BertLayer.NAMES}
        layers.append(BertLayer(cfg, proj, ln))
    tokens = torch.randn((batch, seq, h), generator=_gen(dev, seed + 1), device=dev)
    return BertEncoder(cfg, layers), tokens
