"""Seeded synthetic inputs for the BASELINE.json configurations.

No public suite is involved: BASELINE names synthetic FP64 tensors only.
Two generators produce the same *distribution*:

* ``config0_x`` / ``config1_pair`` -- NumPy, bit-reproducible from a seed,
  used for parity tests and golden fixtures (the oracle sees exactly these
  bits);
* ``config0_x_torch`` / ``config1_pair_torch`` -- the same recipe with
  torch's device RNG, used by ``bench.py`` so large inputs are produced in
  HBM without a host round trip.

Config 0 (BASELINE.json configs[0]): 90% N(0,1); a seeded 10% subset set to
the exact FP64 midpoint between the two FP32 neighbours of its draw, times
(1 + u*2^-40), u ~ U(-1, 1).  Config 1 adds the auditor tensor: the trainer
tensor with a seeded 5% subset moved one FP64 ulp up or down.

``TAU_CONFIG0`` is the reference-form threshold for "1e-3 of the FP32
half-ulp from the midpoint":
tau_ref = 2^-24 - 1e-3 * 2^-24 = 0x1.ff7ced916872bp-25.
"""

from __future__ import annotations

import numpy as np

TAU_CONFIG0 = float.fromhex("0x1.ff7ced916872bp-25")
MID_FRACTION = 0.10
AUDITOR_NOISE_FRACTION = 0.05


def _fp32_bracket(v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """FP32 neighbours (lo <= v <= hi, lo < hi) of FP64 values, as FP64."""
    f = v.astype(np.float32)
    fd = f.astype(np.float64)
    up = np.nextafter(f, np.float32(np.inf)).astype(np.float64)
    dn = np.nextafter(f, np.float32(-np.inf)).astype(np.float64)
    lo = np.where(fd <= v, fd, dn)
    hi = np.where(fd <= v, up, fd)
    return lo, hi


def config0_x(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    k = int(round(MID_FRACTION * n))
    sel = rng.choice(n, size=k, replace=False) if k else np.zeros(0, np.int64)
    u = rng.uniform(-1.0, 1.0, size=k)
    lo, hi = _fp32_bracket(x[sel])
    mid = (lo + hi) * 0.5
    x[sel] = mid * (1.0 + u * 2.0 ** -40)
    return x


def config1_pair(n: int, seed: int = 1) -> tuple[np.ndarray, np.ndarray]:
    x = config0_x(n, seed)
    rng = np.random.default_rng(seed + 1000)
    k = int(round(AUDITOR_NOISE_FRACTION * n))
    sel = rng.choice(n, size=k, replace=False) if k else np.zeros(0, np.int64)
    sgn = rng.integers(0, 2, size=k)
    xa = x.copy()
    xa[sel] = np.nextafter(x[sel], np.where(sgn == 1, np.inf, -np.inf))
    return x, xa


def resnet50_tensors(batch: int = 32, image: int = 224) -> list[tuple[str, tuple[int, ...]]]:
    """The 161 FP64 tensors of BASELINE configs[2]: the 107
    conv / BN / fc forward outputs and the 54 conv / fc input gradients of
    one ResNet-50 step (bottleneck blocks [3, 4, 6, 3], widths 64..512,
    expansion 4, stride on the 3x3 conv), NCHW shapes."""
    fwd: list[tuple[str, tuple[int, ...]]] = []
    grads: list[tuple[str, tuple[int, ...]]] = []

    def conv(name, cin, cout, h, stride, k):
        ho = (h + 2 * (k // 2) - k) // stride + 1
        grads.append((f"grad_in:{name}", (batch, cin, h, h)))
        fwd.append((f"out:{name}", (batch, cout, ho, ho)))
        fwd.append((f"out:{name}.bn", (batch, cout, ho, ho)))
        return ho

    h = conv("conv1", 3, 64, image, 2, 7)
    h = (h + 2 - 3) // 2 + 1  # max pool 3x3 / 2
    cin = 64
    for li, (blocks, width) in enumerate(zip((3, 4, 6, 3), (64, 128, 256, 512))):
        for b in range(blocks):
            stride = 2 if (b == 0 and li > 0) else 1
            name = f"layer{li + 1}.{b}"
            h1 = conv(f"{name}.conv1", cin, width, h, 1, 1)
            h2 = conv(f"{name}.conv2", width, width, h1, stride, 3)
            conv(f"{name}.conv3", width, 4 * width, h2, 1, 1)
            if b == 0:
                conv(f"{name}.downsample", cin, 4 * width, h, stride, 1)
            cin, h = 4 * width, h2
    grads.append(("grad_in:fc", (batch, cin)))
    fwd.append(("out:fc", (batch, 1000)))
    return fwd + grads


def gpt2_small_fp64(device="cuda", vocab: int = 50257, d: int = 768, layers: int = 12, heads: int = 12,
                    ctx: int = 1024, seed: int = 3):
    """BASELINE configs[3] model: GPT-2 small (117M: 12 layers, d=768, 12
    heads, vocab 50257) in FP64 with random init (no checkpoint).  Every
    leaf module is a hook point: wte, wpe, and per block ln_1, c_attn,
    c_proj, ln_2, c_fc, gelu, c_fc_proj; then ln_f and lm_head (tied to wte).
    Attention itself is the functional causal SDPA."""
    import torch
    import torch.nn as nn
    import torch.nn.functional as F

    class Block(nn.Module):
        def __init__(self):
            super().__init__()
            self.ln_1 = nn.LayerNorm(d)
            self.c_attn = nn.Linear(d, 3 * d)
            self.c_proj = nn.Linear(d, d)
            self.ln_2 = nn.LayerNorm(d)
            self.c_fc = nn.Linear(d, 4 * d)
            self.gelu = nn.GELU(approximate="tanh")
            self.c_fc_proj = nn.Linear(4 * d, d)

        def forward(self, x):
            b, t, _ = x.shape
            q, k, v = self.c_attn(self.ln_1(x)).split(d, dim=2)
            q, k, v = (z.view(b, t, heads, d // heads).transpose(1, 2) for z in (q, k, v))
            a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            x = x + self.c_proj(a.transpose(1, 2).reshape(b, t, d))
            return x + self.c_fc_proj(self.gelu(self.c_fc(self.ln_2(x))))

    class GPT2(nn.Module):
        def __init__(self):
            super().__init__()
            self.wte = nn.Embedding(vocab, d)
            self.wpe = nn.Embedding(ctx, d)
            self.h = nn.ModuleList(Block() for _ in range(layers))
            self.ln_f = nn.LayerNorm(d)
            self.lm_head = nn.Linear(d, vocab, bias=False)
            self.lm_head.weight = self.wte.weight

        def forward(self, idx):
            pos = torch.arange(idx.shape[1], device=idx.device)
            x = self.wte(idx) + self.wpe(pos)
            for blk in self.h:
                x = blk(x)
            return self.lm_head(self.ln_f(x))

    torch.manual_seed(seed)
    m = GPT2()
    for name, p in m.named_parameters():
        if name.endswith("weight") and p.dim() == 2:
            torch.nn.init.normal_(p, 0.0, 0.02)
    m = m.to(device=device, dtype=torch.float64)
    m.lm_head.weight = m.wte.weight  # keep the GPT-2 weight tying after the move
    return m


def config2_sigmas(n_tensors: int, seed: int = 2) -> np.ndarray:
    """sigma_t = 10^U(-3, 1) per tensor (log-uniform in [1e-3, 10])."""
    return 10.0 ** np.random.default_rng(seed).uniform(-3.0, 1.0, size=n_tensors)


def config2_tensors_torch(device="cuda") -> list:
    """The 161 configs[2] FP64 tensors exactly as bench.py times them: shapes of
    ``resnet50_tensors`` (flattened), x ~ N(0, sigma_t) drawn in order from one
    torch generator seeded 2 on ``device``."""
    import torch
    shapes = resnet50_tensors()
    sig = config2_sigmas(len(shapes))
    g = torch.Generator(device=device)
    g.manual_seed(2)
    return [torch.randn(int(np.prod(s)), dtype=torch.float64, device=device, generator=g) * float(sig[i])
            for i, (_, s) in enumerate(shapes)]


def config2_budgets(sizes) -> list[int]:
    """B_t = floor(0.005 n_t)."""
    return [int(0.005 * int(n)) for n in sizes]


CONFIG4_PARAMS = 1_500_000_000
CONFIG4_BLOCK = 1 << 22  # parameters per generation block = 16 MiB = one 2^12-leaf Merkle block


def config4_weights_torch(n: int = CONFIG4_PARAMS, device="cuda", lo: int = 0, hi: int | None = None):
    """configs[4]: FP32 weights ~ N(0, 0.02), parameters [lo, hi) of n.  Each
    block of CONFIG4_BLOCK parameters has its own torch generator (seed
    4 << 32 | block), so a rank that owns whole Merkle blocks (dist.
    leaf_block_range, 4 KiB leaves) generates exactly its part of the same
    checkpoint."""
    import torch
    hi = n if hi is None else hi
    if lo % CONFIG4_BLOCK or (hi != n and hi % CONFIG4_BLOCK):
        raise ValueError("lo / hi must be block aligned")
    out = torch.empty(hi - lo, device=device)
    g = torch.Generator(device=device)
    for b0 in range(lo, hi, CONFIG4_BLOCK):
        b1 = min(hi, b0 + CONFIG4_BLOCK)
        g.manual_seed((4 << 32) | (b0 // CONFIG4_BLOCK))
        torch.randn(b1 - b0, device=device, generator=g, out=out[b0 - lo:b1 - lo])
    return out.mul_(0.02)


def _torch_bracket(v):
    import torch
    f = v.float()
    fd = f.double()
    up = torch.nextafter(f, torch.full_like(f, float("inf"))).double()
    dn = torch.nextafter(f, torch.full_like(f, float("-inf"))).double()
    lo = torch.where(fd <= v, fd, dn)
    hi = torch.where(fd <= v, up, fd)
    return lo, hi


def config0_x_torch(n: int, seed: int = 0, device="cuda"):
    """Same recipe as ``config0_x`` drawn with torch's RNG on ``device``
    (not bit-identical to the NumPy stream; used for timing)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(n, dtype=torch.float64, device=device, generator=g)
    k = int(round(MID_FRACTION * n))
    if k:
        sel = torch.randperm(n, device=device, generator=g)[:k]
        u = torch.rand(k, dtype=torch.float64, device=device, generator=g) * 2.0 - 1.0
        lo, hi = _torch_bracket(x[sel])
        x[sel] = (lo + hi) * 0.5 * (1.0 + u * 2.0 ** -40)
    return x


def config0_x_torch_bernoulli(n: int, seed: int = 0, device="cuda"):
    """Config-0 distribution with an i.i.d. 10% midpoint mask instead of an
    exact-size subset (no randperm; used for the 2^20..2^32 size sweep)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(n, dtype=torch.float64, device=device, generator=g)
    chunk = 1 << 26
    for lo in range(0, n, chunk):
        xs = x[lo:lo + chunk]
        m = torch.rand(xs.numel(), device=device, generator=g) < MID_FRACTION
        u = torch.rand(xs.numel(), dtype=torch.float64, device=device, generator=g) * 2.0 - 1.0
        lo_, hi_ = _torch_bracket(xs)
        xs.copy_(torch.where(m, (lo_ + hi_) * 0.5 * (1.0 + u * 2.0 ** -40), xs))
    return x


def config1_pair_torch(n: int, seed: int = 1, device="cuda"):
    import torch
    x = config0_x_torch(n, seed, device)
    g = torch.Generator(device=device)
    g.manual_seed(seed + 1000)
    k = int(round(AUDITOR_NOISE_FRACTION * n))
    xa = x.clone()
    if k:
        sel = torch.randperm(n, device=device, generator=g)[:k]
        sgn = torch.randint(0, 2, (k,), device=device, generator=g)
        tgt = torch.where(sgn == 1, torch.full((k,), float("inf"), dtype=torch.float64, device=device),
                          torch.full((k,), float("-inf"), dtype=torch.float64, device=device))
        xa[sel] = torch.nextafter(x[sel], tgt)
    return x, xa
