# launch list of one HE step (B images) + full captures of the listed kernels, exported to CSV on the box
# usage: bash tools/gpu_profile.sh B "regex1 regex2 ..."
cd $GRAFT_REPO_ROOT
B=${1:-8}; KS=${2:-"ks_inner moddown"}
CMD="python tools/profile_step.py --batch $B"
$CMD > gpurun_out/plain.log 2>&1 || { cat gpurun_out/plain.log; exit 1; }
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_b$B.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
python profiles/summarize_launches.py gpurun_out/launches_b$B.csv | head -30
i=0
for k in $KS; do
  i=$((i+1))
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$k" -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-1} -o /tmp/prof_$i $CMD > gpurun_out/ncu_full_$i.log 2>&1; echo "ncu $k rc=$?"
  ncu -i /tmp/prof_$i.ncu-rep --page raw --csv > gpurun_out/full_$i.csv
  ncu -i /tmp/prof_$i.ncu-rep --page source --csv > gpurun_out/source_$i.csv 2>/dev/null
done
