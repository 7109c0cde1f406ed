# parity tests on the default build, then an interleaved A/B of the bench across variant builds
# usage: bash tools/gpu_ab.sh "variantA variantB" [pytest-args]
cd $GRAFT_REPO_ROOT
VARIANTS="$1"; shift
timeout 1500 python -m pytest tests -m gpu -x -q ${@} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.jsonl').read().strip().splitlines()[-1])
print('main', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'ks frac', round(d['roofline']['frac'],3), 'ntt frac', round(d['roofline_ntt']['frac'],3), d['clocks'])
PY
for rep in 1 2; do
  for v in main $VARIANTS; do
    if [ $v = main ]; then LBL=""; else LBL=$v; fi
    LB_LIB=$LBL timeout 600 python bench.py --no-extras > gpurun_out/bench_$v.jsonl 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_$v.jsonl').read().strip().splitlines()[-1]);print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['reasons'])"
  done
done
