#!/bin/bash
# Round-2d evidence on the GPU box (run from the repo root; outputs in gpurun_out/prof2d/):
#   launch list of the bench's timed steps (gpu__time_duration only) and ncu --set full of the
#   int8 K1, the proposal pack, the L z GEMM, the accept and the cooperative weight update, each
#   captured inside the bench.
set -x
mkdir -p gpurun_out/prof2d
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-path --no-c1 --profile"
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof2d/launches.csv $B > gpurun_out/prof2d/ncu_launches.log 2>&1
full() {  # name regex
  $NCU --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" --launch-skip 3 --launch-count 1 -o gpurun_out/prof2d/$1 $B > gpurun_out/prof2d/ncu_$1.log 2>&1
}
full k1 k1_i8_pair
full pack pack_eps_rows
full lz lz_pair
full accept rw_accept_kernel
$NCU --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:reweight_finish --launch-count 1 -o gpurun_out/prof2d/rwf $B > gpurun_out/prof2d/ncu_rwf.log 2>&1
