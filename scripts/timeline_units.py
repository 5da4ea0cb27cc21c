"""Dev tool: in-kernel timeline of the second-generation kernel on SHORT units (N = 256: four key tiles per unit): clk per
stamp of softmax warp 0, to see what a unit costs beyond its tiles."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ["BA_TC2_MIN_N"] = "128"
import paper_2603_09582_b200 as pkg
H, N, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ba = pkg.BinaryAttention(torch.device("cuda:0"))
Q, K, V = (torch.randn(1, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(3):
    ba.forward(Q, K, V)
Tl = torch.zeros(2 * 148, 4, 256, dtype=torch.int64, device="cuda")
ba.lib.ba_debug_tcgen05_timeline.argtypes = [C.c_void_p]
ba.lib.ba_debug_tcgen05_timeline(C.c_void_p(Tl.data_ptr()))
ba.forward(Q, K, V); torch.cuda.synchronize()
ba.lib.ba_debug_tcgen05_timeline(None)
tl = Tl.cpu().numpy()
T = (N + 63) // 64
if len(sys.argv) > 4 and sys.argv[4] == "epi":  # build with -DBA_DEV_TL_EPI: 4 more stamps per unit (epilogue start, P.V retired, l known, O stored)
    for cta in (0, 74):
        st = tl[cta, 0]; st = st[st > 0]
        per = 5 * T + 4
        n = len(st) // per
        s = st[: n * per].reshape(n, per)
        print(f"=== CTA {cta}: {n} units; per unit: clk from the last tile's P store -> [epilogue start, P.V retired, l exchanged, O stored] -> next unit's first stamp; unit length")
        for u in range(n - 1):
            e = s[u, 5 * T:]
            print(f"  unit {u}: {int(e[0] - s[u, 5 * T - 1])} {int(e[1] - e[0])} {int(e[2] - e[1])} {int(e[3] - e[2])} {int(s[u + 1, 0] - e[3])}   unit {int(s[u + 1, 0] - s[u, 0])}")
    sys.exit(0)
for cta in (0, 74):
    st = tl[cta, 0]; st = st[st > 0]
    n = len(st) // 5
    s = st[: n * 5].reshape(n, 5)
    print(f"=== CTA {cta}: {n} tiles stamped, {T} tiles per unit; rows = units, columns = per-tile [top->S ready, ld issue, ld wait, max, exp+store] then st/loop gap to next stamp")
    for u in range(min(n // T, 6)):
        row = []
        for j in range(T):
            i = u * T + j
            ph = [s[i, 1] - s[i, 0], s[i, 2] - s[i, 1], s[i, 3] - s[i, 2], s[i, 4] - s[i, 3], (s[i + 1, 0] - s[i, 4]) if i + 1 < n else -1]
            row.append("/".join(str(int(x)) for x in ph))
        print(f"  unit {u} ({int(s[u * T, 0] - s[0, 0])} clk): " + "   ".join(row))
    for r, nm in ((1, "mma A"),):
        x = tl[cta, r]; x = x[x > 0]
        print(f"   {nm}: diffs[0:48] {' '.join(str(int(v)) for v in np.diff(x)[:48])}")
