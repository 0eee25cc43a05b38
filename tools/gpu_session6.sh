# TMA-staged P1 lift: parity + probes (MB=3 default, MB=2 variant)
timeout 300 python tools/probe_solve.py C1,C4 auto > gpurun_out/p6_quick.jsonl 2> gpurun_out/p6_quick.err
echo quick rc=$?
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/p6_pytest.log
timeout 600 python tools/probe_solve.py C1,C2,C5,C3,C4 auto > gpurun_out/p6_probe_mb3.jsonl 2> gpurun_out/p6_probe_mb3.err
EGS_LIB=build/libegs_b200_mb2.so timeout 600 python tools/probe_solve.py C1,C2,C5,C3,C4 auto > gpurun_out/p6_probe_mb2.jsonl 2> gpurun_out/p6_probe_mb2.err
cat gpurun_out/p6_pytest.log; tail -n 3 gpurun_out/p6_quick.err gpurun_out/p6_probe_mb3.err
