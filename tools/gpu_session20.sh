EGS_VERBOSE=1 timeout 120 python tools/ncu_target.py C4 2 > gpurun_out/p20_verbose.txt 2>&1; echo rc=$?
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/p20_bench.json 2> gpurun_out/p20_bench.err; echo bench rc=$?
cat gpurun_out/p20_verbose.txt | grep egs
