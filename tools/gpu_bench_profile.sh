# bench + launch list + ncu full captures of k_solve (C4, C3) + a 2-rank
# staged run of the partitioned path; run from the repo root under gpurun
set -u
OUT=gpurun_out/$1
mkdir -p $OUT
sha256sum paper_1710_03647_b200/libegs_b200.so > $OUT/lib_sha256.txt
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/ncu_target.py C4 1 > $OUT/launches.out 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $OUT/solve_c4 python tools/ncu_target.py C4 1 > $OUT/ncu.out 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $OUT/solve_c3 python tools/ncu_target.py C3 1 > $OUT/ncu_c3.out 2>&1; echo "ncu c3 rc=$?"
EGS_BENCH_STAGED=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/bench_2rank_staged.json 2> $OUT/bench_2rank_staged.err; echo "2-rank rc=$?"
cat $OUT/bench.json
