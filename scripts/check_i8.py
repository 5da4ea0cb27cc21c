"""Dev tool: quantize_pv = true on the tensor cores (I8 mode of the second-generation kernel) against the CUDA-core kernel
and the fp64 restatement of attention.cpp:306-363, plus timings of both."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)


def ref_qpv(Q, K, V, bias, scale, bc=64):
    """fp64 restatement of the reference's quantize_pv = true path, one head at a time."""
    B, H, N, d = Q.shape
    out = torch.empty(B, H, N, d, dtype=torch.float64, device=Q.device)
    for b in range(B):
        for h in range(H):
            q, k, v = Q[b, h].double(), K[b, h].double(), V[b, h].double()
            mu = q.abs().mean() * k.abs().mean()
            s = mu * (torch.where(q >= 0, 1.0, -1.0).double() @ torch.where(k >= 0, 1.0, -1.0).double().T) * scale
            if bias is not None:
                s = s + bias[h % bias.shape[0]].double()
            vmax = v.abs().amax(dim=0)
            delta = torch.where(vmax > 0, vmax / 127.0, torch.ones_like(vmax))
            vq = torch.sign(v / delta) * torch.floor((v / delta).abs() + 0.5)
            m = torch.full((N,), -float("inf"), dtype=torch.float64, device=Q.device)
            l = torch.zeros(N, dtype=torch.float64, device=Q.device)
            O = torch.zeros(N, d, dtype=torch.float64, device=Q.device)
            for j0 in range(0, N, bc):
                sb = s[:, j0:j0 + bc]
                m_new = torch.maximum(m, sb.amax(dim=1))
                r = torch.exp(m - m_new)
                p = torch.exp(sb - m_new[:, None])
                l = l * r + p.sum(dim=1)
                p8 = torch.floor(p * 255.0 + 0.5)
                O = O * r[:, None] + p8 @ vq[j0:j0 + bc]
                m = m_new
            out[b, h] = O / l[:, None] / 255.0 * delta[None, :]
    return out


mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode in ("all", "check"):
    for (B, H, N, d, wb) in [(1, 2, 128, 64, False), (1, 2, 256, 64, True), (2, 3, 197, 64, True), (1, 2, 577, 64, False),
                             (1, 2, 1024, 32, False), (1, 2, 512, 48, True), (1, 3, 320, 16, True), (1, 2, 2048, 64, True),
                             (1, 2, 256, 72, True), (2, 2, 1024, 72, False), (1, 2, 384, 128, True), (1, 2, 577, 96, False), (1, 2, 130, 104, True)]:
        Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
        bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
        scale = 1.0 / d ** 0.5
        ref = ref_qpv(Q, K, V, bias, scale)
        o1 = ba.forward(Q, K, V, bias, kernel="simt", quantize_pv=True)
        o2, m2, l2 = ba.forward(Q, K, V, bias, kernel="tcgen05", quantize_pv=True, return_stats=True)
        _, m1, l1 = ba.forward(Q, K, V, bias, kernel="simt", quantize_pv=True, return_stats=True)
        torch.cuda.synchronize()
        e1 = (o1.double() - ref).abs().max().item()
        e2 = (o2.double() - ref).abs().max().item()
        print(f"B{B} H{H} N{N} d{d} bias={wb}: max|O-ref| cuda-core {e1:.2e}  tensor-core {e2:.2e}  |tc-cc| {(o1 - o2).abs().max().item():.2e}"
              f"  stats dm {(m1 - m2).abs().max().item():.1e} dl/l {((l1 - l2).abs() / l1).max().item():.1e}  nan={bool(torch.isnan(o2).any())}", flush=True)
if mode in ("all", "time"):
    for (B, H, N, d) in [(256, 12, 197, 64), (64, 12, 577, 64), (32, 16, 1024, 72), (1, 16, 4096, 64), (1, 16, 4096, 128), (1, 16, 16384, 64)]:
        Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
        bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
        res = {}
        for name, kw in (("bf16 P.V", dict()), ("i8 tensor-core", dict(quantize_pv=True, kernel="tcgen05")), ("i8 cuda-core", dict(quantize_pv=True, kernel="simt"))):
            if name == "i8 cuda-core" and N > 4096:
                continue
            for _ in range(2):
                ba.forward(Q, K, V, bias, **kw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record()
            for _ in range(reps):
                ba.forward(Q, K, V, bias, **kw)
            e1.record(); torch.cuda.synchronize()
            res[name] = e0.elapsed_time(e1) / reps
        print(f"B{B} H{H} N{N} d{d} bias: " + "   ".join(f"{k} {v:.3f} ms" for k, v in res.items()), flush=True)
if mode == "k1v":
    for (B, H, N, d) in [(256, 12, 197, 64), (64, 12, 577, 64), (1, 16, 4096, 64)]:
        V = torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16)
        for _ in range(2):
            ba.quantize_values(V)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ba.quantize_values(V)
        e1.record(); torch.cuda.synchronize()
        print(f"B{B} H{H} N{N} d{d}: quantize_values {e0.elapsed_time(e1) / 10:.3f} ms (includes the output allocations)", flush=True)
