# round-2 profile set: one-step launch list at B=64 + full captures of the
# key-switch kernels (tools/gpu_profile.sh), full captures of the hot-path
# u32 NTT launches (tools/ntt_launch.py), the integer-pipe cross-check
cd $GRAFT_REPO_ROOT
python tools/pipes.py > gpurun_out/r02_pipes.json 2>&1
bash tools/gpu_profile.sh 64 "ks_inner_planes moddown ntt_inverse_kernel" > gpurun_out/prof64.log 2>&1; echo "profile rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:ntt_" -c 2 -o /tmp/prof_ntt python tools/ntt_launch.py > gpurun_out/ncu_ntt.log 2>&1; echo "ncu ntt rc=$?"
ncu -i /tmp/prof_ntt.ncu-rep --page raw --csv > gpurun_out/full_ntt.csv
ncu -i /tmp/prof_ntt.ncu-rep --page source --csv > gpurun_out/source_ntt.csv 2>/dev/null
tail -25 gpurun_out/prof64.log
