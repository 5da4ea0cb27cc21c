#!/bin/bash
# Dev tool: A/B timing of prebuilt library variants (variants/<name>.so, git-ignored) on one box, alternating between them so
# that clock / power-cap drift hits all alike.  usage: scripts/ab.sh ROUNDS SCRIPT v0 v1 [v2 ...]   (SCRIPT: time_bias.py, time_small.py)
R=$1; S=$2; shift; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    cp variants/$v.so paper_2603_09582_b200/libbinattn_cuda.so  # (variants/ is scratch: build each variant with BA_NVCC_FLAGS, copy the .so there; keep it under a few hundred MB -- it travels with gpurun)
    echo "== $v (round $r)"
    timeout 300 python scripts/$S 2>&1 | sed 's/^/   /'
  done
done
