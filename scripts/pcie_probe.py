"""Dev tool: what the host link gives -- H2D alone, D2H alone, both at once (pinned buffers, 256 MB each)."""
import time, torch
n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda"); d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
for _ in range(2): run(True, True)
a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D alone {n/a/1e9:.1f} GB/s   D2H alone {n/b/1e9:.1f} GB/s   both at once: {n/c/1e9:.1f} GB/s each direction ({2*n/c/1e9:.1f} total)")
