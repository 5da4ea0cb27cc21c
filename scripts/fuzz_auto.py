"""Dev tool: random shapes / dtypes / bias forms through kernel="auto" against the CUDA-core kernel (<= 2e-3 in the fp mode, <= 1e-3
in the integer mode), plus NaN checks.  Catches dispatch mistakes at the borders between the kernels."""
import random, sys
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
torch.manual_seed(0)
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 150):
    B, H = random.choice([(1, 1), (1, 2), (2, 3), (1, 5)])
    N = random.choice([1, 2, 7, 31, 63, 64, 65, 100, 127, 128, 129, 196, 197, 255, 256, 257, 400, 511, 512, 513, 600, 1023, 1024, 1100, 2047, 2048, 2049])
    d = random.choice([1, 5, 8, 16, 24, 32, 40, 64, 72, 96, 104, 128, 130, 192, 256])
    dt = random.choice([torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.float16, torch.float32])
    kind = random.choice(["none", "dense", "dense_contig", "dense_f32", "shared", "rel1d", "rel2d"])
    qpv = random.random() < 0.3
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(dt) for _ in range(3))
    bias = None
    if kind == "dense":
        bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    elif kind == "dense_contig":
        bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16)
    elif kind == "dense_f32":
        bias = 0.5 * torch.randn(H, N, N, device="cuda")
    elif kind == "shared":
        bias = (0.5 * torch.randn(1, N, N, device="cuda")).to(torch.bfloat16)
    elif kind == "rel1d":
        bias = pkg.Relative1dBias((0.5 * torch.randn(H, 2 * N - 1, device="cuda")).to(torch.bfloat16))
    elif kind == "rel2d":
        g = int(round(N ** 0.5))
        if g * g != N:
            continue
        bias = pkg.Relative2dBias((0.5 * torch.randn(H, 2 * g - 1, device="cuda")).to(torch.bfloat16), (0.5 * torch.randn(H, 2 * g - 1, device="cuda")).to(torch.bfloat16))
    try:
        a = ba.forward(Q, K, V, bias, quantize_pv=qpv)
        b = ba.forward(Q, K, V, bias, quantize_pv=qpv, kernel="simt")
    except Exception as ex:  # noqa: BLE001
        print(f"B{B} H{H} N{N} d{d} {dt} {kind} qpv={qpv}: EXCEPTION {type(ex).__name__}: {str(ex)[:120]}", flush=True)
        bad += 1
        continue
    e = (a - b).abs().max().item() if a.numel() else 0.0
    tol = 1e-3 if qpv else 2e-3
    if e > tol or bool(torch.isnan(a).any()):
        bad += 1
        print(f"B{B} H{H} N{N} d{d} {dt} {kind} qpv={qpv}: auto-vs-simt {e:.2e}  <-- BAD", flush=True)
print("cases with a problem:", bad)
