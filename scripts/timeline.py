"""Dev tool: dump the in-kernel clock64 timeline of a few CTAs of the (persistent) tcgen05 kernel."""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

B, H, N, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 12, 197, 64))]
use_bias = (sys.argv[5] == "1") if len(sys.argv) > 5 else True
ST = 256
ba = pkg.BinaryAttention(torch.device("cuda:0"))
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if use_bias else None
units = B * H * ((N + 127) // 128)
ctas = min(units, 2 * torch.cuda.get_device_properties(0).multi_processor_count)
NST = int(sys.argv[6]) if len(sys.argv) > 6 else 64
for _ in range(3):
    ba.forward(Q, K, V, bias, kernel="tcgen05")
Tl = torch.zeros(ctas, 4, ST, dtype=torch.int64, device="cuda")
ba.lib.ba_debug_tcgen05_timeline.argtypes = [C.c_void_p]
ba.lib.ba_debug_tcgen05_timeline(C.c_void_p(Tl.data_ptr()))
ba.forward(Q, K, V, bias, kernel="tcgen05"); torch.cuda.synchronize()
ba.lib.ba_debug_tcgen05_timeline(None)
tl = Tl.cpu().numpy()
names = {0: "softmax", 1: "mma", 2: "tma", 3: "expander"}
for cta in [0, ctas // 2]:
    t0 = tl[cta][tl[cta] > 0].min()
    print(f"=== CTA {cta}  (cycles since CTA start; {units} units over {ctas} CTAs)")
    for r in range(4):
        st = tl[cta, r]; st = st[st > 0] - t0
        print(f"  {names[r]:9s} abs  ", " ".join(str(int(x)) for x in st[:NST]))
        print(f"  {names[r]:9s} diff ", " ".join(str(int(x)) for x in np.diff(st[:NST])))
