mkdir -p gpurun_out
(time python -m pytest tests -m gpu -x -q -p no:cacheprovider) > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/fs_probe.py 26 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"fs_" -c 8 -o gpurun_out/fs_full python tools/fs_probe.py 26 > gpurun_out/fs_ncu.log 2>&1; echo "ncu fs rc=$?"
python tools/dct_probe.py 65536 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fast_dct_stream_tr -s 1 -c 1 -o gpurun_out/dct_t_full python tools/dct_probe.py 65536 2 > gpurun_out/dct_t_ncu.log 2>&1; echo "ncu dct_t rc=$?"
