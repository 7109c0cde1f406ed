# round-end measurement set: default bench line, other workloads, reference arm
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_mnist.jsonl 2> gpurun_out/bench_mnist.err; echo "mnist rc=$?"
python bench.py --workload lola-small --no-extras > gpurun_out/bench_small.jsonl 2>/dev/null; echo "small rc=$?"
python bench.py --workload lola-cifar --batch 1 --steps 1 --warmup 3 --no-extras > gpurun_out/bench_cifar.jsonl 2>/dev/null; echo "cifar rc=$?"
python bench.py --workload cryptonets-simd --steps 2 --warmup 3 --no-extras > gpurun_out/bench_simd.jsonl 2>/dev/null; echo "simd rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.jsonl 2>/dev/null; echo "ref rc=$?"
for f in mnist small cifar simd ref; do python -c "
import json;d=json.loads(open('gpurun_out/bench_$f.jsonl').read().strip().splitlines()[-1])
print('$f', d.get('value'), d.get('e2e',{}).get('value') if isinstance(d.get('e2e'),dict) else None, d.get('config',{}).get('workload'), d.get('clocks',{}).get('reasons'))"; done
