# full ncu captures of the key-switch kernels (one launch each) on a short bench run;
# exported to CSV on the box (the reports themselves are too large to bring back)
cd $GRAFT_REPO_ROOT
CMD="python bench.py --batch 8 --steps 1 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
for k in ${KERNELS:-ks_inner moddown ntt_inverse_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o /tmp/prof_$k $CMD > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/full_$k.csv
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv > gpurun_out/source_$k.csv 2>/dev/null
  ls -la /tmp/prof_$k.ncu-rep
done
