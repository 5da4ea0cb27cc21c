"""Dev tool: run-to-run identity of the dense-bias variants of the second-generation kernel, with the location of any difference."""
import os, sys, torch
sys.path.insert(0, ".")
os.environ["BA_TC2_MIN_N_BIAS"] = "512"
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 150
SH = [(2, 16, 2048, 128), (1, 16, 4096, 128), (2, 16, 2048, 64), (4, 16, 1024, 128), (8, 16, 512, 128), (2, 16, 2048, 96), (32, 16, 1024, 72)]
if len(sys.argv) > 2:
    SH = [tuple(int(x) for x in a.split(",")) for a in sys.argv[2:]]
for (B, H, N, d) in SH:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16)
    ref = None
    bad = 0
    where = []
    for i in range(reps):
        o = ba.forward(Q, K, V, bias)
        torch.cuda.synchronize()
        if ref is None:
            ref = o.clone()
        else:
            diff = (o - ref).abs()
            if diff.max().item() != 0.0:
                bad += 1
                if len(where) < 3:
                    idx = (diff.amax(dim=-1) > 0).nonzero()
                    b_, h_ = idx[0, 0].item(), idx[0, 1].item()
                    rows = idx[(idx[:, 0] == b_) & (idx[:, 1] == h_)][:, 2]
                    cols = (diff[b_, h_, rows[0]] > 0).nonzero().flatten()
                    where.append(f"(b{b_} h{h_} rows {rows.min().item()}..{rows.max().item()} n={len(rows)} of {len(idx)} bad rows; cols {cols.min().item()}..{cols.max().item()} n={len(cols)}; max {diff.max().item():.2e})")
    print(f"B{B} H{H} N{N} d{d}: {bad}/{reps - 1} runs differ  {' '.join(where)}", flush=True)
