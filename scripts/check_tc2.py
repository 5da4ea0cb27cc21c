"""Dev tool: second-generation K2 (attn_tc2) against the first-generation kernel and the fp64 torch restatement, plus
timings of both on the long-sequence shapes.  BA_TC2=0/1 switches the dispatch inside the library (read at every call)."""
import os, sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)


def ref64(Q, K, V, bias, scale):
    q, k, v = Q.double(), K.double(), V.double()
    mu = q.abs().mean(dim=(-2, -1), keepdim=True) * k.abs().mean(dim=(-2, -1), keepdim=True)
    sq = torch.where(q >= 0, 1.0, -1.0).double()
    sk = torch.where(k >= 0, 1.0, -1.0).double()
    s = mu * (sq @ sk.transpose(-1, -2)) * scale
    if bias is not None:
        s = s + bias.double()
    return torch.softmax(s, dim=-1) @ v


def run(tc2, *args, **kw):
    os.environ["BA_TC2"] = "1" if tc2 else "0"
    out = ba.forward(*args, **kw)
    torch.cuda.synchronize()
    return out


def timeit(tc2, Q, K, V, bias, reps=20):
    os.environ["BA_TC2"] = "1" if tc2 else "0"
    for _ in range(3):
        ba.forward(Q, K, V, bias)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ba.forward(Q, K, V, bias)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode in ("all", "check"):
    for (B, H, N, d, wb) in [(1, 2, 256, 64, False), (1, 2, 256, 64, True), (2, 3, 384, 72, True), (1, 2, 512, 128, False),
                             (1, 2, 512, 128, True), (1, 4, 1024, 72, True), (1, 2, 640, 32, False), (1, 2, 192, 64, True), (1, 3, 320, 128, False), (1, 2, 2048, 96, True),
                             (1, 6, 577, 64, True), (1, 6, 513, 64, False), (2, 3, 700, 72, True), (1, 2, 833, 128, False), (1, 2, 1000, 96, True), (2, 2, 1023, 64, True), (1, 2, 639, 32, False)]:
        Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
        bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
        scale = 1.0 / d ** 0.5
        ref = ref64(Q, K, V, bias, scale)
        o1 = run(False, Q, K, V, bias)
        o2 = run(True, Q, K, V, bias)
        e1 = (o1.double() - ref).abs().max().item()
        e2 = (o2.double() - ref).abs().max().item()
        o3, rmax, rsum = run(True, Q, K, V, bias, return_stats=True)
        e3 = (o3.double() - ref).abs().max().item()
        print(f"B{B} H{H} N{N} d{d} bias={wb}: max|O-ref| gen1 {e1:.2e}  tc2 {e2:.2e}  tc2+stats {e3:.2e}  nan={bool(torch.isnan(o2).any())}", flush=True)
if mode in ("all", "time"):
    for (B, H, N, d) in [(1, 16, 4096, 64), (1, 16, 4096, 128), (1, 16, 8192, 64), (1, 16, 8192, 128), (1, 16, 16384, 64),
                         (1, 16, 16384, 128), (32, 16, 1024, 72)]:
        Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
        for wb in (False, True):
            bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
            t1 = timeit(False, Q, K, V, bias, 10)
            t2 = timeit(True, Q, K, V, bias, 10)
            tops = 4.0 * B * H * N * N * d / (t2 * 1e-3) / 1e12
            print(f"B{B} H{H} N{N} d{d} bias={wb}: gen1 {t1:.3f} ms  tc2 {t2:.3f} ms  ({t1 / t2:.2f}x, {tops:.0f} eff. TOPS)", flush=True)
            del bias
