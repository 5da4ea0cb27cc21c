"""Dev tool: per-phase clock64 timeline of the second-generation kernel's softmax warp 0 (5 stamps per key tile: tile top,
S load issued, bias + S landed, max agreed, P stored) and of its MMA / producer warps.  Needs a build with the TL variants
(no-bias: always there for d = 64 / 128; dense bias: BA_NVCC_FLAGS=-DBA_DEV_TL_BIAS, d = 128)."""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

H, N, d = [int(x) for x in sys.argv[1:4]]
use_bias = sys.argv[4] == "1"
ST = 256
ba = pkg.BinaryAttention(torch.device("cuda:0"))
Q, K, V = (torch.randn(1, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16) if use_bias else None
for _ in range(3):
    ba.forward(Q, K, V, bias)
Tl = torch.zeros(2 * 148, 4, ST, dtype=torch.int64, device="cuda")
ba.lib.ba_debug_tcgen05_timeline.argtypes = [C.c_void_p]
ba.lib.ba_debug_tcgen05_timeline(C.c_void_p(Tl.data_ptr()))
ba.forward(Q, K, V, bias); torch.cuda.synchronize()
ba.lib.ba_debug_tcgen05_timeline(None)
tl = Tl.cpu().numpy()
names = ["top->S ready (sfull wait)", "S load issue", "bias ready + S landed", "bias add + max + agreement", "exp + pack + P store issue"]
for cta in (0, 74):
    st = tl[cta, 0]; st = st[st > 0]
    n = len(st) // 5
    if n < 12:
        print("no stamps (variant without timeline?)"); break
    s = st[: n * 5].reshape(n, 5)
    ph = np.zeros((n - 1, 5))
    ph[:, 0] = s[:-1, 1] - s[:-1, 0]
    ph[:, 1] = s[:-1, 2] - s[:-1, 1]
    ph[:, 2] = s[:-1, 3] - s[:-1, 2]
    ph[:, 3] = s[:-1, 4] - s[:-1, 3]
    ph[:, 4] = s[1:, 0] - s[:-1, 4]
    lab = ["sfull wait", "S ld issue + bfull wait + ld wait", "bias add + max + agreement", "exp + pack + P store issue", "st wait + fence + arrive + loop"]
    print(f"=== CTA {cta}: {n} tiles stamped; tile period mean {np.diff(s[8:, 0]).mean():.0f} clk (tiles 8..)")
    for i in range(5):
        print(f"   {lab[i]:36s} mean {ph[8:, i].mean():7.0f}  median {np.median(ph[8:, i]):7.0f}  max {ph[8:, i].max():7.0f}")
    for r, nm in ((1, "mma A"), (2, "mma B"), (3, "producer")):
        x = tl[cta, r]; x = x[x > 0]
        if len(sys.argv) > 5 and sys.argv[5] == "mma8" and r < 3:  # build with -DBA_DEV_TL_MMA: 8 stamps per iteration from the second on
            dd = np.diff(x)[6 + 8 * 4: 6 + 8 * 28].reshape(-1, 8)
            lab8 = ["kfull->elect", "4 S mma", "commit sfull", "commit kfree", "leave elect", "p/v waits", "PV issue block", "loop top+tests"]
            print(f"   {nm}: " + "  ".join(f"{l} {int(v)}" for l, v in zip(lab8, np.median(dd, axis=0))) + f"   (sum {int(np.median(dd, axis=0).sum())})")
        else:
            print(f"   {nm}: stamps {len(x)}, diffs[40:60] {' '.join(str(int(v)) for v in np.diff(x)[40:60])}")
