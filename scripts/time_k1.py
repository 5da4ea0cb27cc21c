"""Dev tool: K1 (sign pack + mu of Q and K) alone on the d = 72 configs, new lane mapping against the old one (BA_PACK_NO_D72)."""
import os, sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B, H, N, d) in [(64, 16, 256, 72), (32, 16, 1024, 72), (8, 16, 197, 72)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    res = {}
    for name in ("old", "new"):
        if name == "old": os.environ["BA_PACK_NO_D72"] = "1"
        else: os.environ.pop("BA_PACK_NO_D72", None)
        ts, k1 = [], []
        for it in range(14):
            flush.zero_()
            ba.profile_begin(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); o = ba.forward(Q, K, V); e1.record(); torch.cuda.synchronize()
            n, a, b = ba.profile_end()
            if it >= 3: ts.append(e0.elapsed_time(e1)); k1.append(a)
        res[name] = (statistics.median(ts), statistics.median(k1), o)
    same = torch.equal(res["old"][2], res["new"][2])
    print(f"B{B} H{H} N{N} d{d}: total old {res['old'][0]:.4f} new {res['new'][0]:.4f} ms   K1 old {res['old'][1]:.4f} new {res['new'][1]:.4f} ms   same O: {same}", flush=True)
