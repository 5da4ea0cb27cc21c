import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(1)
B, H, N, d = 4, 16, 1024, 72
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16)
ref = None
for i in range(400):
    o = ba.forward(Q, K, V, bias); torch.cuda.synchronize()
    if ref is None: ref = o.clone(); continue
    bad = (o != ref)
    if bad.any():
        idx = bad.nonzero()
        bh = (idx[:, 0] * H + idx[:, 1]).unique().tolist()
        rows = idx[:, 2]
        cols = idx[:, 3]
        print(f"run {i}: heads {bh} rows [{rows.min().item()}, {rows.max().item()}] n_rows {rows.unique().numel()} cols [{cols.min().item()}, {cols.max().item()}] n_bad {bad.sum().item()} maxdiff {(o-ref).abs().max().item():.3e}; units {[ (h*4 + r//256) for h in bh for r in rows.unique().tolist()[:1]]}", flush=True)
