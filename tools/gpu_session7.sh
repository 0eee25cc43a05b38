# L2 policies: probe + ncu of the solve kernel (C4), TMA vs no-TMA
timeout 120 python tools/probe_solve.py C1,C4 auto > gpurun_out/p7_probe.jsonl 2> gpurun_out/p7_probe.err; echo probe rc=$?
EGS_NO_TMA=1 timeout 120 python tools/probe_solve.py C4 auto > gpurun_out/p7_probe_notma.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/solve_c4_v2 python tools/ncu_target.py C4 1 > gpurun_out/p7_ncu.out 2>&1; echo ncu rc=$?
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
