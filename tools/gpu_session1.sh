set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python tools/probe_solve.py C1,C2,C5 auto,dense,sparse > gpurun_out/probe_small.jsonl 2> gpurun_out/probe_small.err
timeout 600 python tools/probe_solve.py C3 auto > gpurun_out/probe_c3.jsonl 2> gpurun_out/probe_c3.err
timeout 900 python tools/probe_solve.py C4 auto > gpurun_out/probe_c4.jsonl 2> gpurun_out/probe_c4.err
cat gpurun_out/pytest_gpu.log; cat gpurun_out/probe_*.jsonl; tail -5 gpurun_out/*.err
