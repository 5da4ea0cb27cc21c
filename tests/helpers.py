"""Shared input builders: identical values for the CPU checker (float64) and the CUDA path (device dtype)."""
import numpy as np

from oracle import cpu


def make_head_inputs(port, seed, stream, n, d, bias_scale=None, dtype="bf16"):
    """q,k,v (and bias) drawn like the reference's tests (rng.hpp + oracles.hpp random_dense), rounded to `dtype`.
    Same recipe as oracle/gen_golden.py, so golden cases can be regenerated from (seed, stream)."""
    rng = port.make_rng(seed, stream)
    rnd = {"bf16": cpu.bf16_round, "f32": lambda x: x.astype(np.float32).astype(np.float64),
           "f16": lambda x: x.astype(np.float16).astype(np.float64)}[dtype]
    q, k, v = (rnd(rng.random_dense(n, d)) for _ in range(3))
    bias = rnd(rng.random_dense(n, n, bias_scale)) if bias_scale else None
    return q, k, v, bias


def to_torch(x, dtype, device="cuda"):
    """float64 array holding dtype-representable values -> torch tensor of that dtype (exact)."""
    import torch
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16}[dtype]
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device=device, dtype=tdt)


def words_to_numpy(words):
    """int64 torch tensor holding u64 bit patterns -> numpy uint64."""
    return words.cpu().numpy().view(np.uint64)
