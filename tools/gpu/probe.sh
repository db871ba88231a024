# phase probes of K1P (library rebuilt on the box with -DPR_PART_PROBES; PR_PROBE_FLAGS adds e.g. -DPR_PART_NODM)
export PR_EXTRA_NVCC_FLAGS="-DPR_PART_PROBES $PR_PROBE_FLAGS"
python -c "from paper_2508_08873_b200 import build; build.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 60 python tools/k1p_time.py C4 16384 linear 3 | tail -1
PR_PART_PROF=1 timeout 60 python tools/k1p_time.py C4 16384 linear 1 2>&1 | grep -E "part probes|max active" | tail -2
