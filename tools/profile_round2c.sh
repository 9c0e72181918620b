#!/bin/bash
# Round-2c evidence on the GPU box (run from the repo root; outputs in gpurun_out/prof2c/):
#   launch list of the bench's timed steps (gpu__time_duration only), ncu --set full of the int8
#   K1 kernel inside the bench, of the MwG initialisation chains (K=148, the burn-in layout) and of
#   the lambda-step MwG move kernel.
set -x
mkdir -p gpurun_out/prof2c
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-path --profile"
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof2c/launches.csv $B > gpurun_out/prof2c/ncu_launches.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:k1_i8_pair --launch-skip 3 --launch-count 1 -o gpurun_out/prof2c/k1_full $B \
  > gpurun_out/prof2c/ncu_k1.log 2>&1
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:mwg_kernel \
  --launch-skip 1 --launch-count 1 -o gpurun_out/prof2c/mwg_chain_full python tools/mwg_profile_chain.py 148 4 4 \
  > gpurun_out/prof2c/ncu_mwg.log 2>&1
