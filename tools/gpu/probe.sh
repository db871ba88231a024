# phase probes of K1P (library built with -DPR_PART_PROBES)
export PR_EXTRA_NVCC_FLAGS=-DPR_PART_PROBES
for tm in 0 1; do
  echo "== PR_PART_NOTMEM=$tm"
  PR_PART_NOTMEM=$tm timeout 60 python tools/k1p_time.py C4 16384 linear 3 | tail -1
  PR_PART_NOTMEM=$tm PR_PART_PROF=1 timeout 60 python tools/k1p_time.py C4 16384 linear 1 2>&1 | grep -E "part probes|max active" | tail -2
done
