#!/bin/bash
# Round-2 evidence on the GPU box (run from the repo root; outputs in gpurun_out/prof2/):
#   launch list of the bench command (gpu__time_duration only: the recipe's
#   pass), ncu --set full of K1 and of a live resampling step's kernels.
#   (compute-sanitizer is closed on this pool: see DESIGN.md section 4.)
set -x
mkdir -p gpurun_out/prof2
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/prof2/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-path \
  > gpurun_out/prof2/ncu_launches.log 2>&1
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiSoftplus \
  --launch-skip 6 --launch-count 1 \
  -o gpurun_out/prof2/k1_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-path \
  > gpurun_out/prof2/ncu_k1.log 2>&1
$NCU --set full --clock-control none --import-source on \
  -k regex:"scan_tile_sums|scan_segments|scan_values|ancestors_kernel|peer_gather|resample_commit" \
  --launch-skip 6 --launch-count 6 -o gpurun_out/prof2/resample_full env SPA_NO_PROFILER=1 python tools/resample_micro.py \
  > gpurun_out/prof2/ncu_resample.log 2>&1
