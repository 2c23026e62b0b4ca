#!/usr/bin/env bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   1. the bench line (plain run, no profiler)             -> gpurun_out/bench.json
#   2. the launch list of the same command (cold, serial)  -> gpurun_out/launches.csv
#   3. ncu --set full of the hot kernels of one DLT (split_b, split-int8 GEMM,
#      NDCT) at a reduced column count (same kernels, same N; replay cost
#      bounded)                                           -> gpurun_out/hot_full.ncu-rep
#   4. ncu --set full of the plain DCT-III pass (streaming kernel, 4096 x 65536,
#      the HBM-bound pass of north_star's 60% target)      -> gpurun_out/dct_full.ncu-rep
#   5. ncu --set full of the IDLT's NDCT^T kernel (16384 columns)
#                                                          -> gpurun_out/tr_full.ncu-rep
set -u
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python tools/kernel_probe.py dlt 4096 8192 3 > gpurun_out/kern_small.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"fast_ndct_fwd|oz_gemm2|oz_split_b" -s 3 -c 3 \
    -o gpurun_out/hot_full python tools/kernel_probe.py dlt 4096 8192 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
python tools/dct_probe.py > gpurun_out/dct_probe.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:fast_dct_stream -s 2 -c 1 \
    -o gpurun_out/dct_full python tools/dct_probe.py > gpurun_out/dct_ncu.log 2>&1
echo "ncu dct rc=$?"
python tools/kernel_probe.py ndct_t 4096 16384 2 > gpurun_out/idlt_probe.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:fast_ndct_tr -s 1 -c 1 \
    -o gpurun_out/tr_full python tools/kernel_probe.py ndct_t 4096 16384 2 > gpurun_out/tr_ncu.log 2>&1
echo "ncu tr rc=$?"
