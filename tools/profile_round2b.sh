#!/bin/bash
# Round-2 (int8 K1) evidence on the GPU box (run from the repo root; outputs in gpurun_out/prof2b/):
#   launch list of the bench's timed steps (gpu__time_duration only, --profile-from-start off
#   + bench.py --profile), ncu --set full of the int8 K1 kernel and of the proposal pack.
set -x
mkdir -p gpurun_out/prof2b
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-path --profile"
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof2b/launches.csv $B > gpurun_out/prof2b/ncu_launches.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:k1_i8_pair --launch-skip 3 --launch-count 1 -o gpurun_out/prof2b/k1_full $B \
  > gpurun_out/prof2b/ncu_k1.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:pack_eps --launch-skip 3 --launch-count 1 -o gpurun_out/prof2b/pack_full $B \
  > gpurun_out/prof2b/ncu_pack.log 2>&1
