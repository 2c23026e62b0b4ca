#!/usr/bin/env bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   1. the bench line (plain run, no profiler)             -> gpurun_out/bench.json
#   2. the launch list of the same command (cold, serial)  -> gpurun_out/launches.csv
#   3. ncu --set full of one direct DLT + IDLT (digit splits + dense GEMM) at a
#      reduced column count (same kernels, same N)         -> gpurun_out/direct_full.ncu-rep
#   4. ncu --set full of the factored NDCT / NDCT^T kernels -> gpurun_out/ndct_full.ncu-rep
#   5. ncu --set full of the plain DCT-III pass (streaming kernel, 4096 x 65536,
#      the HBM-bound pass of north_star's 60% target)      -> gpurun_out/dct_full.ncu-rep
set -u
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs \
    > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python tools/kernel_probe.py dlt 4096 8192 2 > gpurun_out/kern_small.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm2|oz_split_b" -s 2 -c 2 \
    -o gpurun_out/direct_full python tools/kernel_probe.py dlt 4096 8192 2 > gpurun_out/ncu_direct.log 2>&1
echo "ncu direct rc=$?"
python tools/kernel_probe.py idlt 4096 8192 2 > gpurun_out/kern_small_i.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"oz_gemm2|oz_split_b_sym" -s 2 -c 2 \
    -o gpurun_out/direct_idlt_full python tools/kernel_probe.py idlt 4096 8192 2 > gpurun_out/ncu_direct_i.log 2>&1
echo "ncu direct idlt rc=$?"
python tools/kernel_probe.py ndct 4096 8192 2 > gpurun_out/kern_ndct.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"fast_ndct" -s 1 -c 1 \
    -o gpurun_out/ndct_full python tools/kernel_probe.py ndct 4096 8192 2 > gpurun_out/ncu_ndct.log 2>&1
echo "ncu ndct rc=$?"
python tools/kernel_probe.py ndct_t 4096 8192 2 > gpurun_out/kern_ndct_t.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"fast_ndct_tr" -s 1 -c 1 \
    -o gpurun_out/ndct_t_full python tools/kernel_probe.py ndct_t 4096 8192 2 > gpurun_out/ncu_ndct_t.log 2>&1
echo "ncu ndct_t rc=$?"
python tools/kernel_probe.py dct 4096 65536 2 > gpurun_out/dct_probe.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:fast_dct_stream -s 1 -c 1 \
    -o gpurun_out/dct_full python tools/kernel_probe.py dct 4096 65536 2 > gpurun_out/dct_ncu.log 2>&1
echo "ncu dct rc=$?"
