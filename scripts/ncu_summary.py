"""Summarise an .ncu-rep (run where ncu is installed; no GPU needed): key raw metrics per kernel + hottest SASS lines.
usage: python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_name.txt"""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg"]


def run(args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rep = sys.argv[1]
rows = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
hdr, units = rows[0], rows[1]
print(f"# ncu summary of {rep} (ncu --set full --clock-control none --import-source on; replayed, cold-cache timings)")
for r in rows[2:]:
    print(f"\n## kernel: {r[hdr.index('Kernel Name')]}")
    for k in KEYS:
        if k in hdr:
            print(f"  {k:72s} {r[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
    mult = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = sum(float(r[hdr.index(k)].replace(",", "")) * mult.get(units[hdr.index(k)], 1.0)
              for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"  {'traffic = dram read + write':72s} {tot / 1e6:16.3f} Mbyte")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv"]))))
if len(src) > 2:
    h = src[1]
    ix = {k: i for i, k in enumerate(h)}
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    data = []
    for r in src[2:]:
        if len(r) < len(h):
            continue
        try:
            data.append((r[ix["Source"]], int(r[ix["Instructions Executed"]] or 0), int(r[ix["# Samples"]] or 0),
                         {s: int(r[ix[s]] or 0) for s in stalls}))
        except ValueError:
            pass
    tot = sum(d[2] for d in data) or 1
    print(f"\n## hottest SASS instructions by warp-stall samples (last profiled kernel; total samples {tot}, total warp instructions {sum(d[1] for d in data)})")
    for s, ex, sm, st in sorted(data, key=lambda t: -t[2])[:20]:
        top = max(st.items(), key=lambda kv: kv[1])
        print(f"  {100*sm/tot:5.1f}%  exec {ex:10d}  {s[:80]:80s} {top[0]}={top[1]}")
    agg = {}
    for s, ex, sm, st in data:
        for k, v in st.items():
            agg[k] = agg.get(k, 0) + v
    print("\n## stall reasons (all samples):", ", ".join(f"{k}={v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
