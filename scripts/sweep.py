"""BASELINE.json metric sweep: BinaryAttention fwd ms / effective TOPS vs the best bf16 dense-attention kernel on the
same GPU, for every config of BASELINE.json (C2..C5).  Writes one JSON object per line.
usage: python scripts/sweep.py [out.jsonl] [--quick]"""
import json, sys, time
import torch
import torch.nn.functional as F
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

out_path = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "gpurun_out/sweep.jsonl"
quick = "--quick" in sys.argv
shapes = [("c2", 256, 12, 197, 64), ("c3", 64, 16, 256, 72), ("c4", 32, 16, 1024, 72), ("c5", 1, 16, 4096, 64),
          ("c5", 1, 16, 4096, 128), ("c5", 1, 16, 8192, 64), ("c5", 1, 16, 8192, 128), ("c5", 1, 16, 16384, 64),
          ("c5", 1, 16, 16384, 128)]
if quick:
    shapes = shapes[:5]
ba = pkg.BinaryAttention(torch.device("cuda:0"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def time_ms(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()  # L2 flush between timed iterations
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def dense_candidates(Q, K, V, bias):
    """bf16 dense attention kernels available in this image; returns {name: callable}."""
    c = {}
    from torch.nn.attention import sdpa_kernel, SDPBackend
    for name, be in (("sdpa_flash", SDPBackend.FLASH_ATTENTION), ("sdpa_cudnn", SDPBackend.CUDNN_ATTENTION),
                     ("sdpa_efficient", SDPBackend.EFFICIENT_ATTENTION)):
        def f(be=be):
            with sdpa_kernel([be]):
                return F.scaled_dot_product_attention(Q, K, V, attn_mask=bias)
        c[name] = f
    if bias is None:
        try:
            from flash_attn import flash_attn_func
            Qt, Kt, Vt = (x.transpose(1, 2).contiguous() for x in (Q, K, V))
            if Q.shape[-1] % 8 == 0:
                c["flash_attn2"] = lambda: flash_attn_func(Qt, Kt, Vt)
        except Exception:
            pass
    return c


with open(out_path, "w") as fo:
    for (tag, B, H, N, d) in shapes:
        Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
        ld = (N + 7) // 8 * 8
        for use_bias in (False, True, "rel1d"):
            if use_bias and H * N * ld * 2 > (12 << 30):
                continue
            bias = None
            ours_bias = None
            if use_bias is True:
                store = torch.empty(H, N, ld, device="cuda", dtype=torch.bfloat16)
                store.normal_(0, 0.5)
                bias = ours_bias = store[:, :, :N]
            elif use_bias == "rel1d":
                # Relative1dBias: ours gets the 2N-1 offsets per head, the dense kernel the N x N table they expand to
                offs = (0.5 * torch.randn(H, 2 * N - 1, device="cuda")).to(torch.bfloat16).float()
                idx = torch.arange(N, device="cuda")[:, None] - torch.arange(N, device="cuda")[None, :] + (N - 1)
                bias = offs[:, idx].to(torch.bfloat16)
                del idx
                ours_bias = pkg.Relative1dBias(offs)
            for _ in range(2):  # warm-up (first call builds tensor maps / sets attributes)
                ba.forward(Q, K, V, ours_bias, kernel="tcgen05")
            ba.profile_begin(4)
            for _ in range(4):
                ba.forward(Q, K, V, ours_bias, kernel="tcgen05")
            torch.cuda.synchronize()
            n, k1, k2 = ba.profile_end()
            ours = time_ms(lambda: ba.forward(Q, K, V, ours_bias, kernel="tcgen05"))
            dense = {}
            dbias = bias.unsqueeze(0).expand(B, H, N, N) if use_bias else None
            for name, fn in dense_candidates(Q, K, V, dbias).items():
                try:
                    dense[name] = time_ms(fn, reps=10)
                except Exception as e:  # backend does not take this shape / mask
                    dense[name] = None
            ok = {k: v for k, v in dense.items() if v}
            best = min(ok, key=ok.get) if ok else None
            ops = 4.0 * B * H * N * N * d
            rec = {"config": tag, "B": B, "H": H, "N": N, "d": d,
                   "bias": {False: "none", True: "dense", "rel1d": "rel1d (ours: 2N-1 offsets; dense: the N x N table)"}[use_bias],
                   "ours_ms": ours,
                   "k1_pack_ms": k1 / n, "k2_attn_ms": k2 / n, "ours_eff_tops": ops / ours / 1e9,
                   "dense_bf16_ms": dense, "dense_best": best, "dense_best_ms": ok.get(best),
                   "dense_best_eff_tops": ops / ok[best] / 1e9 if best else None,
                   "speedup_vs_dense_bf16": ok[best] / ours if best else None,
                   "timing": "median of 20 (ours) / 10 (dense), CUDA events, L2 flushed between iterations"}
            print(json.dumps(rec), flush=True)
            fo.write(json.dumps(rec) + "\n")
            del bias, ours_bias
        del Q, K, V
        torch.cuda.empty_cache()
