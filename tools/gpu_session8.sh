timeout 120 python tools/probe_solve.py C1,C2,C5,C3,C4 auto > gpurun_out/p8_probe.jsonl 2> gpurun_out/p8_probe.err; echo probe rc=$?
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
