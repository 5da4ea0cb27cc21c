"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol include/binattn_cuda.h
declares, status codes behave, the launcher partition is right, and the N>1 host logic works over gloo."""
import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2603_09582_b200 import load_library
    return load_library()


def test_every_declared_symbol_is_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "binattn_cuda.h")).read()
    declared = set(re.findall(r"\b(ba_[a-z_0-9]+)\s*\(", hdr))
    assert {"ba_create", "ba_destroy", "ba_pack_signs", "ba_binary_logits", "ba_binary_attention_fwd",
            "ba_binary_attention_host", "ba_workspace_bytes", "ba_shard_range", "ba_last_error"} <= declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in binattn_cuda.h but not exported"


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = lib.ba_create(0, C.byref(h))
    assert rc == 3 and b"no CPU fallback" in lib.ba_last_error()
    import paper_2603_09582_b200 as pkg
    with pytest.raises(pkg.CudaError):
        pkg.BinaryAttention()
    with pytest.raises(pkg.CudaError):
        pkg.binary_attention(torch.zeros(1, 1, 4, 8), torch.zeros(1, 1, 4, 8), torch.zeros(1, 1, 4, 8))


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure; nothing under the product package may import, link or run it."""
    pkg = os.path.join(ROOT, "paper_2603_09582_b200")
    pat = re.compile(r"(from\s+oracle|import\s+oracle|oracle/|binattn_oracle|libbinattn_ref|bo_[a-z_]+\()")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
                assert not pat.search(open(os.path.join(dp, f)).read()), f"{f} reaches into oracle/"


def test_workspace_and_param_validation(lib):
    from paper_2603_09582_b200.api import _Params
    p = _Params(B=2, H=3, N=197, d=72, in_dtype=0, inv_tau=0.1)
    ws = lib.ba_workspace_bytes(C.byref(p))
    assert ws >= 2 * 2 * 3 * 197 * 2 * 8  # two packed planes of ceil(72/64)=2 u64 per row
    p.N = 0
    assert lib.ba_workspace_bytes(C.byref(p)) == 0


def test_ctypes_mirror_matches_the_header_field_for_field(tmp_path):
    """api._Params must be include/binattn_cuda.h's ba_params: same field names in the same order, same offsets and total
    size (a compiled probe prints offsetof for every field the header declares)."""
    import re
    import subprocess
    from paper_2603_09582_b200.api import _Params
    hdr = open(os.path.join(ROOT, "include", "binattn_cuda.h")).read()
    body = hdr[hdr.index("typedef struct {", hdr.index("ba_bias_mode")):hdr.index("} ba_params;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in re.findall(r"(?:int32_t|int64_t|float)\s+([^;]+);", body):
        names += [n.strip() for n in decl.split(",")]
    assert names == [f[0] for f in _Params._fields_]
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "binattn_cuda.h"\nint main(void){'
                   + "".join(f'printf("%zu\\n", offsetof(ba_params, {n}));' for n in names)
                   + 'printf("%zu\\n", sizeof(ba_params));return 0;}')
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals[:-1] == [getattr(_Params, n).offset for n in names]
    assert vals[-1] == C.sizeof(_Params)


def test_shard_range_matches_python_and_covers(lib):
    from paper_2603_09582_b200 import shard_range
    for total in (0, 1, 6, 16, 512, 3072, 3073):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for rank in range(world):
                b, e = C.c_int64(), C.c_int64()
                assert lib.ba_shard_range(total, world, rank, C.byref(b), C.byref(e)) == 0
                assert (b.value, e.value) == shard_range(total, world, rank)
                covered += list(range(b.value, e.value))
            assert covered == list(range(total))
            sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    b, e = C.c_int64(), C.c_int64()
    assert lib.ba_shard_range(4, 2, 2, C.byref(b), C.byref(e)) == 2  # ValidationError
    # (head, 256-row block) units: B*H*ceil(N/256) of them, same arithmetic
    from paper_2603_09582_b200.api import _Params
    lib.ba_shard_units.argtypes = [C.POINTER(_Params), C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    p = _Params(B=1, H=16, N=4096, d=64)
    got = []
    for rank in range(8):
        assert lib.ba_shard_units(C.byref(p), 8, rank, C.byref(b), C.byref(e)) == 0
        assert (b.value, e.value) == shard_range(16 * 16, 8, rank)
        got.append((b.value, e.value))
    assert got[0][0] == 0 and got[-1][1] == 256 and all(got[i][1] == got[i + 1][0] for i in range(7))


def test_reference_error_mirrors():
    import torch
    from paper_2603_09582_b200 import AttentionConfig, binary_attention_fused, ShapeError, ValidationError
    cfg = AttentionConfig.make(4, 3)
    assert cfg.temperature == pytest.approx(3 ** 0.5) and cfg.block_rows == 4
    q, bad = torch.zeros(4, 3), torch.zeros(4, 2)
    with pytest.raises(ShapeError):  # test_attention.cpp:134-136
        binary_attention_fused(q, q, bad, cfg)
    big = AttentionConfig.make(4, 3)
    big.block_rows = 9
    with pytest.raises(ValidationError):  # test_attention.cpp:137-139
        binary_attention_fused(q, q, q, big)
    neg = AttentionConfig.make(4, 3)
    neg.temperature = 0.0
    with pytest.raises(ValidationError):
        binary_attention_fused(q, q, q, neg)


_GLOO_WORKER = r"""
import os, sys
sys.path.insert(0, os.environ["BA_ROOT"])
import numpy as np, torch, torch.distributed as dist
from paper_2603_09582_b200 import shard_range, shard_heads
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
B, H, N, d = 3, 5, 7, 4
x = torch.arange(B * H * N * d, dtype=torch.float32).reshape(B, H, N, d)
mine = shard_heads(x, world, rank)                       # this rank's heads, no data-path collective
b, e = shard_range(B * H, world, rank)
assert mine.shape == (1, e - b, N, d)
out = mine * 2.0 + 1.0                                   # stand-in for the per-head kernel (heads independent)
# verification-only gather (outside any timed region in bench.py): ragged shards -> pad to the max count
counts = [shard_range(B * H, world, r)[1] - shard_range(B * H, world, r)[0] for r in range(world)]
pad = torch.zeros(1, max(counts), N, d); pad[:, : e - b] = out
bufs = [torch.zeros_like(pad) for _ in range(world)]
dist.all_gather(bufs, pad)
full = torch.cat([bufs[r][:, : counts[r]] for r in range(world)], dim=1).reshape(B, H, N, d)
assert torch.equal(full, x * 2.0 + 1.0), "1-vs-k shard gather mismatch"
# the launcher class (same plan / gather code bench.py runs under torchrun with NCCL), batch-split and head-split plans
from paper_2603_09582_b200 import ShardedBinaryAttention, shard_plan, shard_units
sh = ShardedBinaryAttention(rank, world, 0)
for (Bb, Hh) in ((4, 3), (1, 5), (3, 5)):
    xb = torch.arange(Bb * Hh * N * d, dtype=torch.float32).reshape(Bb, Hh, N, d)
    bias = torch.arange(Hh * N * N, dtype=torch.float32).reshape(Hh, N, N)
    Ql, Kl, Vl, bl = sh.shard(xb, xb, xb, bias)
    pl = shard_plan(Bb, Hh, world, rank)
    assert Ql.shape[0] * Ql.shape[1] == pl["end"] - pl["begin"]
    if pl["mode"] == "heads" and Ql.shape[1]:  # one bias table per local head, in grid order
        assert bl.shape[0] == Ql.shape[1] and torch.equal(bl[0], bias[pl["begin"] % Hh])
    assert torch.equal(sh.gather(Ql * 3.0, Bb, Hh), xb * 3.0)
# (head, 256-row block) units: the ranks' ranges tile the grid, and a rank's rows are the rows of its units
ranges = [shard_units(1, 5, 600, world, r) for r in range(world)]
assert ranges[0][0] == 0 and ranges[-1][1] == 5 * 3 and all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
t = torch.tensor([float(rank + 1)]); dist.all_reduce(t, op=dist.ReduceOp.MAX)   # max-over-ranks timing reduction
assert t.item() == world
dist.barrier(); dist.destroy_process_group()
print("OK", rank)
"""


def test_two_rank_gloo_shard_and_gather(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(_GLOO_WORKER)
    env = dict(os.environ, BA_ROOT=ROOT, MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29631", str(script)],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("OK") == 2
