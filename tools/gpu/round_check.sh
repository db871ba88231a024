# full GPU check of a round: GPU tests, default bench, ncu launch list of the bench command,
# one full ncu capture of the dominant kernel (K1P, C4 LINEAR launch)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-sub > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_step -s 1 -c 1 -o gpurun_out/r2_k1p_tm_c4 -f python tools/k1p_once.py C4 16384 > gpurun_out/ncu_k1p.log 2>&1
ncu -i gpurun_out/r2_k1p_tm_c4.ncu-rep --page raw --csv > gpurun_out/r2_k1p_tm_c4_raw.csv 2>/dev/null
tail -3 gpurun_out/gputest.log
