"""Dev tool: forward() per call with an L2 flush between calls (median/min) and back to back, for a few long shapes
(used to find the programmatic-launch regression at 3.46 units per CTA; BA_PDL=0/1 overrides the policy)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B,H,N,d) in [(1,16,8192,64),(1,16,8192,128),(1,16,4096,64),(1,16,16384,64)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    for _ in range(3): ba.forward(Q, K, V)
    ts=[]
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ba.forward(Q, K, V); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ba.forward(Q, K, V)
    e1.record(); torch.cuda.synchronize()
    print(f"N{N} d{d}: flushed median {ts[10]*1e3:.1f} us min {ts[0]*1e3:.1f}; back-to-back {e0.elapsed_time(e1)/20*1e3:.1f} us")
