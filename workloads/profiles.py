"""Seeded synthetic layer profiles — the ONLY module shared by `oracle/` and the CUDA path.

It holds none of the method's arithmetic: it only produces per-layer forward/backward
milliseconds F[l][d], B[l][d] (d = 1..M GPUs of one node, stored at column d-1) and
per-layer model-state bytes, with the shapes and value distributions of the paper's
workloads (PAPER.md `tab:models` P:661-676, layer counts P:819).  The recipe is the one
stated in SURVEY.md §8(d) and restated in DESIGN.md §"Input recipe".

Randomness is a counter-based generator (splitmix64 of (seed, stream, index)), so any
value can be regenerated independently of call order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """One splitmix64 output for state x (Steele et al.); pure integer bit mixing."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def uniform(seed: int, stream: int, index: int) -> float:
    """Counter-based U[0,1) with 53 random bits, keyed by (seed, stream, index)."""
    key = splitmix64((seed * 0x100000001B3) & MASK64)
    key = splitmix64(key ^ ((stream * 0xD6E8FEB86659FD93) & MASK64))
    r = splitmix64(key ^ (index & MASK64))
    return (r >> 11) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, index: int) -> float:
    """Box-Muller standard normal from two counter-based uniforms."""
    u1 = uniform(seed, stream, 2 * index)
    u2 = uniform(seed, stream, 2 * index + 1)
    u1 = max(u1, 1e-300)
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def dyadic(x: float, bits: int = 20) -> float:
    """Round to a multiple of 2^-bits (>= 2^-bits) so sums/products stay exact."""
    q = float(1 << bits)
    return max(round(x * q), 1) / q


@dataclass
class Profile:
    """Per-layer costs: fwd_ms/bwd_ms are float64 [L][M] (column d-1 = d GPUs)."""
    name: str
    fwd_ms: np.ndarray
    bwd_ms: np.ndarray
    state_bytes: np.ndarray
    act_bytes: np.ndarray = field(default=None)

    @property
    def L(self) -> int:
        return int(self.fwd_ms.shape[0])

    @property
    def M(self) -> int:
        return int(self.fwd_ms.shape[1])


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config: L layers, M GPUs/node, N nodes, f, n0 (explicit)."""
    key: str
    label: str
    L: int
    M: int
    N: int
    f: int
    n0: int
    hidden: int = 0
    seq: int = 2048
    microbatch: int = 1
    num_profiles: int = 1
    seed: int = 1

    @property
    def n_max(self) -> int:
        # sizes n0 .. min(N - f*n0, L)  (capped at L: DESIGN reading R4)
        return min(self.N - self.f * self.n0, self.L)


CONFIGS = {
    "cfg1": Config("cfg1", "GPT-2-small-shaped 12-layer, N=4x1 GPU, f=1", 12, 1, 4, 1, 1,
                   hidden=768, seq=1024, microbatch=8, seed=101),
    "cfg2": Config("cfg2", "GPT-3 1.3B-shaped 24-layer, N=16x4 GPUs, f=2", 24, 4, 16, 2, 1,
                   hidden=2048, seq=2048, microbatch=4, seed=102),
    "cfg3": Config("cfg3", "GPT-3 6.7B-shaped 32-layer, N=64x8 GPUs, f=3", 32, 8, 64, 3, 1,
                   hidden=4096, seq=2048, microbatch=2, seed=103),
    "cfg4": Config("cfg4", "GPT-3 175B-shaped 96-layer, N=512x8 GPUs, f=4", 96, 8, 512, 4, 3,
                   hidden=12288, seq=2048, microbatch=1, seed=104),
    "cfg5": Config("cfg5", "batched sweep: 1024 random 48-layer profiles, N=128x8, f=2",
                   48, 8, 128, 2, 1, num_profiles=1024, seed=5000),
}

# tab:planning_latency: one template of n nodes x M GPUs for 24/32/64/96
# layers.  The paper names the 24-layer (BERT-Large, GPT-2, GPT-3 Medium) and 32-layer
# (GPT-3 2.7B/6.7B) models; the 64- and 96-layer profiles are not described, so the
# grid uses GPT-shaped profiles of hidden size 1024 / 2560 / 8192 / 12288.
PLANNING_GRID_LAYERS = {24: 1024, 32: 2560, 64: 8192, 96: 12288}
PLANNING_GRID_NODES = (8, 16, 24)
PLANNING_GRID_GPUS = (1, 4, 8)
PLANNING_GRID_PAPER_S = {   # seconds, [nodes][gpus] -> (24, 32, 64, 96 layers)
    (8, 1): (0.28, 0.71, 9.65, 68.50), (8, 4): (0.41, 1.15, 11.58, 74.56), (8, 8): (0.54, 1.50, 20.98, 109.76),
    (16, 1): (3.37, 7.45, 66.35, 540.36), (16, 4): (4.56, 10.41, 108.10, 649.67),
    (16, 8): (4.90, 11.78, 176.04, 1213.63), (24, 1): (11.35, 30.11, 262.47, 1477.54),
    (24, 4): (14.78, 45.80, 472.53, 2153.84), (24, 8): (15.59, 49.25, 520.08, 3297.92)}


def planning_grid_config(L: int, nodes: int, M: int) -> "Config":
    """The grid point as a Config: one template of `nodes` nodes (n0 = nodes, f = 0, N = nodes)."""
    return Config(f"grid-L{L}-n{nodes}-g{M}", f"tab:planning_latency {L} layers, {nodes} nodes x {M} GPUs",
                  L, M, nodes, 0, nodes, hidden=PLANNING_GRID_LAYERS[L], seq=2048, microbatch=1, seed=200 + L)


VOCAB = 50257
ASSUMED_TFLOPS = 400e12   # per-GPU effective throughput used to turn FLOPs into ms
TP_EFF = 0.85             # SPEC S:61 synth formula fwd[d] = fwd[1] / (1 + eff*(d-1))


def gpt_profile(cfg: Config, seed: int | None = None, mode: str = "real") -> Profile:
    """GPT-shaped profile (cfg1-4): block FLOPs 24bsh^2 + 4bs^2h, LM head on the last layer."""
    seed = cfg.seed if seed is None else seed
    b, s, h, L, M = cfg.microbatch, cfg.seq, cfg.hidden, cfg.L, cfg.M
    fwd = np.empty((L, M), dtype=np.float64)
    bwd = np.empty((L, M), dtype=np.float64)
    for l in range(L):
        flops = 24.0 * b * s * h * h + 4.0 * b * s * s * h
        if l == L - 1:
            flops += 2.0 * b * s * h * VOCAB
        if l == 0:
            flops *= 1.005
        jitter = 1.0 + 0.02 * (uniform(seed, 1, l) - 0.5)
        f1 = flops / ASSUMED_TFLOPS * 1e3 * jitter
        for d in range(1, M + 1):
            fd = f1 / (1.0 + TP_EFF * (d - 1))
            bd = 2.0 * fd
            if mode == "dyadic":
                fd, bd = dyadic(fd), dyadic(bd)
            fwd[l, d - 1] = fd
            bwd[l, d - 1] = bd
    state = np.full(L, 16 * 12 * h * h, dtype=np.int64)
    act = np.full(L, 34 * s * h, dtype=np.int64)
    return Profile(f"{cfg.key}-seed{seed}-{mode}", fwd, bwd, state, act)


def random_profile(seed: int, L: int, M: int, kind: str = "lognormal", mode: str = "real") -> Profile:
    """Random per-layer profile (cfg5 recipe for kind='lognormal'; small-test kinds too).

    kinds: 'lognormal' (cfg5: 10ms*LogN(0,0.35), 10% heavy x U[2,6], bwd = fwd*U[1.8,2.4],
    TP efficiency eta~U[0.6,0.95]); 'uniform' (U[0.5,1.5]); 'integer' (integers 1..9, exact);
    'spiky' (mostly 1, some 20); 'constant' (all layers equal, massive ties).
    """
    fwd = np.empty((L, M), dtype=np.float64)
    bwd = np.empty((L, M), dtype=np.float64)
    eta = 0.6 + 0.35 * uniform(seed, 2, 0)
    for l in range(L):
        if kind == "lognormal":
            f1 = 10.0 * math.exp(0.35 * normal(seed, 3, l))
            if uniform(seed, 4, l) < 0.1:
                f1 *= 2.0 + 4.0 * uniform(seed, 5, l)
            r = 1.8 + 0.6 * uniform(seed, 6, l)
        elif kind == "uniform":
            f1 = 0.5 + uniform(seed, 3, l)
            r = 2.0
        elif kind == "integer":
            f1 = float(1 + int(uniform(seed, 3, l) * 9))
            r = 2.0
        elif kind == "spiky":
            f1 = 20.0 if uniform(seed, 3, l) < 0.2 else 1.0
            r = 2.0
        elif kind == "constant":
            f1 = 2.0
            r = 2.0
        else:
            raise ValueError(kind)
        for d in range(1, M + 1):
            if kind in ("integer", "spiky", "constant"):
                # exact small integers / halves: every sum and product is exact
                fd = f1 if d == 1 else float(max(1, int(f1 / (1.0 + 0.5 * (d - 1)))))
                bd = r * fd
            else:
                fd = f1 / (1.0 + eta * (d - 1))
                bd = r * fd
                if mode == "dyadic":
                    fd, bd = dyadic(fd), dyadic(bd)
            fwd[l, d - 1] = fd
            bwd[l, d - 1] = bd
    state = np.full(L, 1 << 28, dtype=np.int64)
    return Profile(f"rand-{kind}-{seed}-L{L}M{M}-{mode}", fwd, bwd, state)


def costs_profile(costs, M: int = 1, name: str = "costs") -> Profile:
    """Profile whose per-layer F+B equals the given costs exactly (F = B = c/2, exact in
    binary64 for integer c), identical for every d in 1..M."""
    c = np.asarray(costs, dtype=np.float64)
    L = c.shape[0]
    fwd = np.zeros((L, M), dtype=np.float64)
    bwd = np.zeros((L, M), dtype=np.float64)
    for d in range(M):
        fwd[:, d] = c / 2.0
        bwd[:, d] = c / 2.0
    return Profile(name, fwd, bwd, np.full(L, 1 << 20, dtype=np.int64))


def config_profiles(cfg: Config, mode: str = "real", count: int | None = None) -> list[Profile]:
    """The profile(s) of a BASELINE config. cfg5 yields `count` (default 1024) random ones."""
    if cfg.key == "cfg5":
        n = cfg.num_profiles if count is None else count
        return [random_profile(cfg.seed + i, cfg.L, cfg.M, "lognormal", mode) for i in range(n)]
    n = 1 if count is None else count
    return [gpt_profile(cfg, cfg.seed + 1000 * i, mode) for i in range(n)]


def unif6() -> Profile:
    """SPEC S:64 fixture UNIF6: 6 identical layers, fwd 2 ms, bwd 4 ms, M = 1."""
    fwd = np.full((6, 1), 2.0)
    bwd = np.full((6, 1), 4.0)
    return Profile("UNIF6", fwd, bwd, np.full(6, 10 ** 8, dtype=np.int64))
