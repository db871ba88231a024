# cluster occupancy / global exchange microbenchmark, then K1P TM with the interface off (timing aid)
timeout 60 ./tools/ub/ub_clusters > gpurun_out/ub_clusters.txt 2>&1; echo "rc=$?"
for ni in 0 1; do
  PR_PART_NOIFACE=$ni timeout 60 python tools/k1p_time.py C4 16384 linear 5 2>&1 | tail -1 | sed "s/^/noiface=$ni /"
done | tee gpurun_out/noiface.txt
