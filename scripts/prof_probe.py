"""Dev tool: per-call K2 time from the C ABI's profiling events against plain per-call event timing (default bench workload)."""
import sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
B, H, N, d = 1, 16, 16384, 128
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16)
for _ in range(5):
    ba.forward(Q, K, V, bias)
torch.cuda.synchronize()
plain, k1s, k2s = [], [], []
for it in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ba.forward(Q, K, V, bias); e1.record(); torch.cuda.synchronize()
    plain.append(e0.elapsed_time(e1))
for it in range(20):
    ba.profile_begin(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ba.forward(Q, K, V, bias); e1.record(); torch.cuda.synchronize()
    n, k1, k2 = ba.profile_end()
    k1s.append(k1); k2s.append(k2); plain.append(-e0.elapsed_time(e1))
print("plain per-call ms      :", " ".join(f"{x:.3f}" for x in plain[:20]))
print("profiled call total ms :", " ".join(f"{-x:.3f}" for x in plain[20:]))
print("profiled K1 ms         :", " ".join(f"{x:.3f}" for x in k1s))
print("profiled K2 ms         :", " ".join(f"{x:.3f}" for x in k2s))
ba.profile_begin(20)
for _ in range(20):
    ba.forward(Q, K, V, bias)
torch.cuda.synchronize()
print("20 back to back, profiled:", ba.profile_end())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ba.forward(Q, K, V, bias)
e1.record(); torch.cuda.synchronize()
print("20 back to back, plain ms per step:", e0.elapsed_time(e1) / 20)
