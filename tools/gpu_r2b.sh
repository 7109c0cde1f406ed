# round-2b iteration: correctness subset, then A/B of runtime switches on one box
# usage: bash tools/gpu_r2b.sh "<env-assignments-A>|<env-assignments-B>|..." [reps] [tests]
cd $GRAFT_REPO_ROOT
TESTS=${3:-"tests/test_bfv_gpu.py tests/test_sweep_batch_gpu.py tests/test_lola_gpu.py"}
if [ "$TESTS" != none ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -x -q > gpurun_out/r2b_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2b_tests.txt
fi
IFS='|' read -ra VARS <<< "$1"
for rep in $(seq 1 ${2:-2}); do
  for v in "${VARS[@]}"; do
    k=$(env $v timeout 300 python tools/kbench.py 2>&1 | tail -1)
    env $v timeout 600 python bench.py --no-extras > gpurun_out/bench_ab.jsonl 2>gpurun_out/bench_ab.err
    b=$(python -c "import json;d=json.loads(open('gpurun_out/bench_ab.jsonl').read().strip().splitlines()[-1]);print(round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'], d['parity']['mismatches'])" 2>&1 | tail -1)
    echo "[$v] | $k | $b"
  done
done
