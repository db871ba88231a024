# quick K1P check: launch times, then the 1D fine-solve parity tests (short timeouts: a hung
# cluster kernel must not eat the GPU budget)
for mode in linear offset affine; do
  timeout 60 python tools/k1p_time.py C4 16384 $mode 5 2>&1 | tail -1
  echo "rc=$?"
done
timeout 400 python -m pytest tests/test_gpu_1d.py -x -q --timeout 120 -k "fine_linear_adjoint or bitwise or persistent or affine_offset" 2>&1 | tail -3
