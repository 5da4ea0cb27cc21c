#!/bin/bash
# Round-2 evidence capture on one B200 (run under gpurun): bench lines, ncu summaries of the final build, launch list, sanitizer.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err
python bench.py --workload c2 --no-sweep > gpurun_out/r02_bench_c2.json 2>> gpurun_out/r02_bench_default.err
python bench.py --workload c4 --no-sweep > gpurun_out/r02_bench_c4.json 2>> gpurun_out/r02_bench_default.err
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
$NCU -k regex:attn_tc2 -o gpurun_out/r02_c5_16384_128_bias python scripts/run_one.py 1 16 16384 128 1 3 > gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_c5_16384_128_nobias python scripts/run_one.py 1 16 16384 128 0 3 >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_c5_16384_64_nobias python scripts/run_one.py 1 16 16384 64 0 3 >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_c5_16384_64_bias python scripts/run_one.py 1 16 16384 64 1 3 >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_i8_c5_16384_64_bias python scripts/run_one.py 1 16 16384 64 1 3 qpv >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_i8_c2_bias python scripts/run_one.py 256 12 197 64 1 3 qpv >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_c5_4096_64_nobias python scripts/run_one.py 1 16 4096 64 0 3 >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc2 -o gpurun_out/r02_c4_nobias python scripts/run_one.py 32 16 1024 72 0 3 >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc_kernel -o gpurun_out/r02_c4_bias python scripts/run_one.py 32 16 1024 72 1 3 >> gpurun_out/ncu.log 2>&1
$NCU -k regex:attn_tc_kernel -o gpurun_out/r02_c2_bias python scripts/run_one.py 256 12 197 64 1 3 >> gpurun_out/ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_default.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu-baseline --no-traffic > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_tc2.py tests/test_gpu_i8_tc.py tests/test_gpu_out_dtype.py -q -m gpu -k "matches_oracle or logits or unit_shards or fast_path or matches_reference_default or dispatch or rounded_fp32" > gpurun_out/r02_sanitizer_memcheck.txt 2>&1
tail -5 gpurun_out/r02_sanitizer_memcheck.txt
python scripts/peakedness_table.py > gpurun_out/r02_peakedness.md 2>&1
python scripts/check_i8.py time > gpurun_out/r02_i8_times.txt 2>&1
for f in gpurun_out/r02_*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>/dev/null; done
# (gpurun merges at most 64 MiB back: the summaries travel, of the reports only the headline kernel's and the I8 one)
for f in gpurun_out/r02_*.ncu-rep; do case $f in *c5_16384_128_bias*|*i8_c2_bias*) ;; *) rm -f $f;; esac; done
ls -la gpurun_out | tail -20
