# bench + launch list + one full ncu capture of the lift kernel (C4)
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_target.py C4 1 > gpurun_out/ncu_launch.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lift -s 1 -c 2 -o gpurun_out/lift_c4 python tools/ncu_target.py C4 1 > gpurun_out/ncu_full.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cert_prune -c 1 -o gpurun_out/cert_c4 python tools/ncu_target.py C4 1 > gpurun_out/ncu_cert.out 2>&1
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err gpurun_out/ncu_full.out
