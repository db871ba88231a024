# quick K1P check: launch times (TMEM variant and PR_PART_NOTMEM=1), then the 1D fine-solve parity tests
for mode in linear offset affine; do
  PR_PART_NOTMEM=0 timeout 60 python tools/k1p_time.py C4 16384 $mode 5 2>&1 | tail -1 | sed "s/^/NOTMEM=0 /"
  echo "rc=$?"
done
PR_PART_NOTMEM=0 timeout 60 python tools/k1p_time.py C2 2560 linear 5 2>&1 | tail -1
PR_PART_NOTMEM=0 timeout 60 python tools/k1p_time.py C2 20480 linear 5 2>&1 | tail -1
PR_PART_NOTMEM=1 timeout 60 python tools/k1p_time.py C2 20480 linear 5 2>&1 | tail -1 | sed "s/^/NOTMEM=1 /"
timeout 400 python -m pytest tests/test_gpu_1d.py -x -q --timeout 120 -k "fine_linear_adjoint or bitwise or persistent or affine_offset" 2>&1 | tail -3
