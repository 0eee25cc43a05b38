# bench + launch list + ncu full capture of k_solve (C4); run from repo root
set -u
OUT=gpurun_out/$1
mkdir -p $OUT
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/ncu_target.py C4 1 > $OUT/launches.out 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o $OUT/solve_c4 python tools/ncu_target.py C4 1 > $OUT/ncu.out 2>&1; echo "ncu rc=$?"
cat $OUT/bench.json
