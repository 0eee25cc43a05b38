# persistent-kernel solver: parity + probes + bench
timeout 300 python tools/probe_solve.py C1 auto > gpurun_out/p3_c1.jsonl 2>&1
echo "c1 rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/p3_pytest.log
echo "pytest rc=$?"
timeout 600 python tools/probe_solve.py C1,C2,C5,C3,C4 auto,dense,sparse > gpurun_out/p3_probe.jsonl 2> gpurun_out/p3_probe.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/p3_bench.json 2> gpurun_out/p3_bench.err
cat gpurun_out/p3_c1.jsonl gpurun_out/p3_pytest.log; tail -n 5 gpurun_out/p3_probe.err gpurun_out/p3_bench.err
