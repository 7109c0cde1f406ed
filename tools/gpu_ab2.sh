# interleaved A/B across variant builds: kernel rooflines (tools/kbench.py) and
# the bench value (--no-extras); usage: bash tools/gpu_ab2.sh "main varA varB" [reps]
cd $GRAFT_REPO_ROOT
for rep in $(seq 1 ${2:-2}); do
  for v in $1; do
    if [ $v = main ]; then LBL=""; else LBL=$v; fi
    k=$(LB_LIB=$LBL timeout 300 python tools/kbench.py 2>&1 | tail -1)
    LB_LIB=$LBL timeout 600 python bench.py --no-extras > gpurun_out/bench_$v.jsonl 2>/dev/null
    b=$(python -c "import json;d=json.loads(open('gpurun_out/bench_$v.jsonl').read().strip().splitlines()[-1]);print(round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'], d['parity']['mismatches'])" 2>&1)
    echo "$v | $k | $b"
  done
done
