# round-end measurement set: GPU tests, the default bench line (with every
# extra leg), the other workloads, and the reference arm on the same box
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02_gpu_tests.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_mnist.jsonl 2> gpurun_out/r02_bench_mnist.err; echo "mnist rc=$?"
python bench.py --workload lola-small --no-extras > gpurun_out/r02_bench_small.jsonl 2>/dev/null; echo "small rc=$?"
python bench.py --workload lola-cifar --steps 2 --warmup 2 --no-extras > gpurun_out/r02_bench_cifar.jsonl 2>/dev/null; echo "cifar rc=$?"
python bench.py --workload cryptonets-simd --steps 2 --warmup 3 --no-extras > gpurun_out/r02_bench_simd.jsonl 2>/dev/null; echo "simd rc=$?"
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.jsonl 2>/dev/null; echo "ref rc=$?"
for f in mnist small cifar simd ref; do python -c "
import json;d=json.loads(open('gpurun_out/r02_bench_$f.jsonl').read().strip().splitlines()[-1])
print('$f', round(d.get('value',0),3), (d.get('e2e') or {}).get('value'), d.get('parity'), d.get('config',{}).get('workload'), (d.get('clocks') or {}).get('reasons'))"; done
