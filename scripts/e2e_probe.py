"""Dev tool: end-to-end (host buffers) time of the default workload for the current BA_HOST_CHUNK_MB."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
B, H, N, d = 256, 12, 197, 64
ba = pkg.BinaryAttention(torch.device("cuda:0"))
Q, K, V = (torch.randn(B, H, N, d).to(torch.bfloat16).pin_memory() for _ in range(3))
bias = (0.5 * torch.randn(H, N, 200)).to(torch.bfloat16)[:, :, :N].contiguous().pin_memory()
out = torch.empty(B, H, N, d, dtype=torch.float32).pin_memory()
for _ in range(3):
    ba.forward_host(Q, K, V, bias, out=out)
ts = []
for _ in range(15):
    t0 = time.perf_counter(); ba.forward_host(Q, K, V, bias, out=out); ts.append(time.perf_counter() - t0)
ts.sort()
print(f"e2e ms: min {ts[0]*1e3:.2f} median {ts[len(ts)//2]*1e3:.2f} max {ts[-1]*1e3:.2f}")
