set -x
python -c "from paper_2508_08873_b200 import build as B; B.build()" > gpurun_out/build.log 2>&1
for mode in linear offset adjoint; do
  timeout 120 python tools/k1p_time.py C4 16384 $mode 5
  PR_PART_NOPERSIST=1 timeout 120 python tools/k1p_time.py C4 16384 $mode 5
done > gpurun_out/k1p_time.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_1d.py -x -q -k "persistent or bitwise or fine_linear_adjoint or affine_offset or parareal" > gpurun_out/t1d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t1d.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-sub > gpurun_out/bench_c4_p.json 2> gpurun_out/bench_c4_p.err
