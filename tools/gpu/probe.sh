export PR_EXTRA_NVCC_FLAGS=-DPR_PART_PROBES
for tm in 1 0; do
  echo "== PR_PART_NOTMEM=$tm"
  PR_PART_NOTMEM=$tm timeout 120 python tools/k1p_time.py C4 16384 linear 3
  PR_PART_NOTMEM=$tm PR_PART_PROF=1 timeout 120 python tools/k1p_time.py C4 16384 linear 1 2>&1 | grep -E "part probes|max active" | tail -2
done
timeout 600 python -m pytest tests/test_gpu_1d.py -x -q -k "fine_linear_adjoint or bitwise" 2>&1 | tail -3
