# bench + launch list + ncu full captures of k_solve (C4, C3) + the
# all-configs table + a 2-rank (one-GPU) run of the partitioned path; run from
# the repo root under gpurun:  bash tools/gpu_bench_profile.sh <tag>
set -u
OUT=gpurun_out/$1
mkdir -p $OUT
sha256sum paper_1710_03647_b200/libegs_b200.so > $OUT/lib_sha256.txt
python -c "import bench; print(bench.source_digest())" > $OUT/source_digest.txt
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/ncu_target.py C4 1 > $OUT/launches.out 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $OUT/solve_c4 python tools/ncu_target.py C4 1 > $OUT/ncu.out 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $OUT/solve_c3 python tools/ncu_target.py C3 1 > $OUT/ncu_c3.out 2>&1; echo "ncu c3 rc=$?"
EGS_TRACE=1 timeout 300 python tools/ncu_target.py C4 1 > $OUT/trace_c4.txt 2>&1
EGS_TRACE=1 timeout 300 python tools/ncu_target.py C3 1 > $OUT/trace_c3.txt 2>&1
timeout 1200 python tools/config_table.py --out $OUT/configs.jsonl > $OUT/configs.out 2>&1; echo "configs rc=$?"
timeout 600 python tools/part_local_bench.py C4 2 > $OUT/part_local_c4.json 2> $OUT/part_local_c4.err; echo "part-local rc=$?"
timeout 300 python tools/e2e_breakdown.py C4 > $OUT/e2e_breakdown.txt 2>&1; echo "e2e rc=$?"
# two processes on the one GPU over CUDA IPC (functional: contexts of two
# processes time-slice the GPU, so the time is not a scaling number)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/bench_2proc_1gpu.json 2> $OUT/bench_2proc_1gpu.err; echo "2proc rc=$?"
timeout 900 python -m pytest tests -m gpu -q > $OUT/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "reference arm rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
cat $OUT/bench.json

