"""Layer-cost profiler on the local B200 (real profile ingestion).

The planner's input is, per layer l and GPU count d = 1..M of one node, the forward and
backward times F_{l,d}, B_{l,d} (PAPER Eq.4: "F_{l,d} ... the forward time of
layer l with d GPUs").  The paper profiles its models before planning (§3.4 step 2); here a
GPT block with random weights (no dataset, no checkpoint: the times do not depend on the
values) is timed with CUDA events for every tensor-parallel degree d:

* d-way tensor parallelism within the node (Megatron layout, the in-stage parallelism the
  paper realises with FSDP): one GPU runs the 1/d shard of the block — ceil(heads/d)
  attention heads (QKV and output projections sliced), ceil(4h/d) MLP columns — and the
  slowest shard sets the time (the shards are equal up to rounding);
* plus the block's all-reduces of b x s x h bf16 activations: 2 in the forward, 2 in the
  backward.  Their time comes from an NCCL all-reduce measured over d GPUs of this node when
  torch.distributed is initialised with >= d ranks (`measure_allreduce`), else from the
  ring model 2 (d-1)/d x bytes / busbw + latency with the caller's bus bandwidth.

Layer 0 adds the token embedding, the last layer the final LayerNorm and the (d-sharded)
LM head.  state_bytes = 16 bytes per parameter (bf16 weight + fp32 master + Adam moments);
activation_bytes_per_sample from the peak memory of one forward.  The output is the SPEC
profile JSON that `oob_load_profile` / `planner.load_profile` read.

Tooling around the hot path, not the hot path: plain PyTorch (cuBLAS / flash attention via
scaled_dot_product_attention) on bf16.
"""
from __future__ import annotations

import json
import math
import statistics

import torch
import torch.nn.functional as F


def _time_ms(fn, reps: int, warmup: int = 3) -> float:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


class _Shard(torch.nn.Module):
    """1/d tensor-parallel shard of a GPT block (pre-LN attention + 4h MLP)."""

    def __init__(self, h: int, heads: int, d: int, dtype):
        super().__init__()
        hd = h // heads
        self.nh = math.ceil(heads / d)
        self.hd = hd
        w = self.nh * hd
        self.ff = math.ceil(4 * h / d)
        self.ln1 = torch.nn.LayerNorm(h, dtype=dtype)
        self.qkv = torch.nn.Linear(h, 3 * w, dtype=dtype)
        self.proj = torch.nn.Linear(w, h, dtype=dtype)
        self.ln2 = torch.nn.LayerNorm(h, dtype=dtype)
        self.fc1 = torch.nn.Linear(h, self.ff, dtype=dtype)
        self.fc2 = torch.nn.Linear(self.ff, h, dtype=dtype)

    def forward(self, x):
        b, s, h = x.shape
        q, k, v = self.qkv(self.ln1(x)).view(b, s, 3, self.nh, self.hd).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + self.proj(a.transpose(1, 2).reshape(b, s, self.nh * self.hd))
        return x + self.fc2(F.gelu(self.fc1(self.ln2(x))))


def measure_allreduce(nbytes: int, group=None, reps: int = 20) -> float:
    """Median ms of one NCCL all-reduce of nbytes (bf16) over `group` (torch.distributed)."""
    import torch.distributed as dist
    t = torch.zeros(nbytes // 2, dtype=torch.bfloat16, device="cuda")
    return _time_ms(lambda: dist.all_reduce(t, group=group), reps)


def allreduce_model_ms(nbytes: int, d: int, busbw_gbps: float, latency_us: float = 8.0) -> float:
    """Ring all-reduce time model: 2 (d-1)/d x bytes / bus bandwidth + latency."""
    if d <= 1:
        return 0.0
    return 2.0 * (d - 1) / d * nbytes / (busbw_gbps * 1e9) * 1e3 + latency_us * 1e-3


def profile_gpt(hidden: int, heads: int, layers: int, seq: int, microbatch: int, gpus_per_node: int,
                vocab: int = 50257, reps: int = 10, allreduce_ms=None, busbw_gbps: float = 0.0,
                dtype=torch.bfloat16) -> dict:
    """SPEC S:99 profile of a GPT model of `layers` blocks measured on this GPU.
    allreduce_ms: optional callable (nbytes, d) -> ms (e.g. measured with measure_allreduce
    over d ranks); else the ring model with busbw_gbps (> 0 required when M > 1)."""
    dev = torch.device("cuda")
    M = gpus_per_node
    act_bytes_ar = microbatch * seq * hidden * 2
    fwd_block, bwd_block, fwd_head, bwd_head = {}, {}, {}, {}
    act_per_sample = 0
    for d in range(1, M + 1):
        torch.manual_seed(d)
        blk = _Shard(hidden, heads, d, dtype).to(dev)
        x = torch.randn(microbatch, seq, hidden, dtype=dtype, device=dev, requires_grad=True)
        gy = torch.randn_like(x)

        def fwd():
            with torch.no_grad():
                blk(x)

        def fwd_bwd():
            y = blk(x)
            y.backward(gy)
        f = _time_ms(fwd, reps)
        fb = _time_ms(fwd_bwd, reps)
        if d == 1:
            torch.cuda.reset_peak_memory_stats()
            base = torch.cuda.memory_allocated()
            y = blk(x)
            act_per_sample = (torch.cuda.max_memory_allocated() - base) // microbatch
            del y
        ar = 0.0
        if d > 1:
            if allreduce_ms is not None:
                ar = allreduce_ms(act_bytes_ar, d)
            elif busbw_gbps > 0:
                ar = allreduce_model_ms(act_bytes_ar, d, busbw_gbps)
            else:
                raise ValueError("M > 1 needs allreduce_ms or busbw_gbps for the tensor-parallel all-reduces")
        fwd_block[d] = f + 2 * ar
        bwd_block[d] = max(fb - f, 1e-6) + 2 * ar
        # LM head (d-sharded vocab projection) + final LayerNorm, on the last layer
        wv = math.ceil(vocab / d)
        head = torch.nn.Linear(hidden, wv, bias=False, dtype=dtype, device=dev)
        xh = torch.randn(microbatch, seq, hidden, dtype=dtype, device=dev, requires_grad=True)
        gh = torch.randn(microbatch, seq, wv, dtype=dtype, device=dev)
        fh = _time_ms(lambda: head(xh).detach(), reps)
        fbh = _time_ms(lambda: head(xh).backward(gh), reps)
        fwd_head[d], bwd_head[d] = fh, max(fbh - fh, 1e-6)
        del blk, x, gy, head, xh, gh
        torch.cuda.empty_cache()
    params_block = 12 * hidden * hidden + 13 * hidden
    out_layers = []
    for l in range(layers):
        f = {str(d): fwd_block[d] for d in range(1, M + 1)}
        b = {str(d): bwd_block[d] for d in range(1, M + 1)}
        params = params_block
        if l == 0:
            params += vocab * hidden + seq * hidden      # token + position embeddings (lookup: no GEMM time)
        if l == layers - 1:
            for d in range(1, M + 1):
                f[str(d)] += fwd_head[d]
                b[str(d)] += bwd_head[d]
        out_layers.append({"name": f"block{l}", "state_bytes": 16 * params,
                           "activation_bytes_per_sample": int(act_per_sample),
                           "fwd_ms": f, "bwd_ms": b})
    return {"gpus_per_node": M, "microbatch_reference": microbatch,
            "measured_on": torch.cuda.get_device_name(), "dtype": str(dtype).replace("torch.", ""),
            "layers": out_layers}


def write_profile(doc: dict, path: str) -> None:
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)          # floats as repr: exact binary64 round trip
