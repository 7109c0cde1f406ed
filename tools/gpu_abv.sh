# interleaved A/B of the bench (no tests) across variant builds, 3 rounds
# usage: bash tools/gpu_abv.sh "variantA variantB"
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  for v in main $1; do
    if [ $v = main ]; then LBL=""; else LBL=$v; fi
    LB_LIB=$LBL timeout 600 python bench.py --no-extras > gpurun_out/bench_$v.jsonl 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_$v.jsonl').read().strip().splitlines()[-1]);print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_min_mhz'])"
  done
done
