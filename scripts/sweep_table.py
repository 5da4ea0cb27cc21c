"""Renders the markdown table of a scripts/sweep.py result.  usage: python scripts/sweep_table.py in.jsonl > out.md"""
import json, sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print("# BASELINE.json metric sweep (round 1, final kernels): BinaryAttention fwd vs the fastest bf16 dense-attention kernel on the same B200\n")
print("Produced by `python scripts/sweep.py` on one B200 (median of 20 / 10 timed runs, CUDA events, L2 flushed between iterations);")
print("table rendered by `scripts/sweep_table.py`.")
print("`ours` = K1 sign-pack+mu + K2 fused attention; `dense` = fastest of torch SDPA cuDNN / flash / efficient backends and flash-attn 2.")
print("bias `dense`: both sides read the same additive N×N bf16 table (only cuDNN and efficient accept one). bias `rel1d`: ours gets the")
print("2N−1 `Relative1dBias` offsets and generates the bias in-kernel, the dense kernel needs the N×N table they expand to.")
print("Effective TOPS = 4·B·H·N²·d / t.\n")
print("| config | B | H | N | d | bias | ours ms (K1 + K2) | ours eff. TOPS | dense best | dense ms | dense eff. TOPS | speedup |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['config']} | {r['B']} | {r['H']} | {r['N']} | {r['d']} | {r['bias']} | {r['ours_ms']:.3f} ({r['k1_pack_ms']:.3f} + {r['k2_attn_ms']:.3f}) | "
          f"{r['ours_eff_tops']:.0f} | {r['dense_best']} | {r['dense_best_ms']:.3f} | {r['dense_best_eff_tops']:.0f} | {r['speedup_vs_dense_bf16']:.2f}x |")
