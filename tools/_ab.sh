B='timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline'
P='import json,sys; d=json.loads(sys.stdin.readline()); k=d["kernels_ms"]; print(round(k["leg2cheb_split_int8"],3), round(k["dlt_step"],3), round(k["idlt_step"],3), d["parity_check"]["rel_err_vs_oracle"])'
for i in 1 2; do
echo -n "pair "; $B 2>/dev/null | python -c "$P"
echo -n "1sm  "; FLB_LIB_PATH=paper_1505_00354_b200/build/variants/lib_1sm.so $B 2>/dev/null | python -c "$P"
done
FLB_LIB_PATH=paper_1505_00354_b200/build/variants/lib_1sm.so timeout 300 python -m pytest tests/test_gpu_int8_split.py -q 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_int8_split.py -q 2>&1 | tail -1
