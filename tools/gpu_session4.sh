# ncu full capture of the persistent solve kernel on C4 + build-step timings
EGS_VERBOSE=1 timeout 300 python tools/ncu_target.py C4 2 > gpurun_out/p4_verbose.txt 2>&1
EGS_VERBOSE=1 timeout 300 python tools/ncu_target.py C3 2 >> gpurun_out/p4_verbose.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/solve_c4 python tools/ncu_target.py C4 1 > gpurun_out/p4_ncu.out 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p4_launches.csv python tools/ncu_target.py C4 1 > /dev/null 2>&1
cat gpurun_out/p4_verbose.txt; tail -3 gpurun_out/p4_ncu.out
