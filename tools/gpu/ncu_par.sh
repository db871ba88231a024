# ncu --set full captures of the Parareal-side HBM kernels (projection k_xty_rm<true>, expansion k_expand_mma)
# from one C4 Parareal run with one iteration
timeout 120 python tools/tools_ncu_par.py 1 > gpurun_out/ncu_par_plain.log 2>&1; echo "plain rc=$?"
for k in k_xty_rm k_expand_mma; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/r2_$k -f python tools/tools_ncu_par.py 1 > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/r2_$k.ncu-rep --page raw --csv > gpurun_out/r2_${k}_raw.csv 2>/dev/null
  echo "$k rc=$?"
done
