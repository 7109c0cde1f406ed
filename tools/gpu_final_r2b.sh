# round-2 end measurement set at the final code: GPU tests, smoke, the default
# bench line (every extra leg), the other workloads, the reference arm, then the
# profile set (launch list of one B=64 step, ncu --set full of the key-switch
# kernels and of the hot-path NTT launches, the integer-pipe cross-check)
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_mnist.jsonl 2> gpurun_out/r02_bench_mnist.err; echo "mnist rc=$?"
python bench.py --workload lola-small --no-extras > gpurun_out/r02_bench_small.jsonl 2>/dev/null; echo "small rc=$?"
python bench.py --workload lola-cifar --steps 2 --warmup 2 --no-extras > gpurun_out/r02_bench_cifar.jsonl 2>/dev/null; echo "cifar rc=$?"
python bench.py --workload cryptonets-simd --steps 2 --warmup 3 --no-extras > gpurun_out/r02_bench_simd.jsonl 2>/dev/null; echo "simd rc=$?"
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.jsonl 2>/dev/null; echo "ref rc=$?"
for f in mnist small cifar simd ref; do python -c "
import json;d=json.loads(open('gpurun_out/r02_bench_$f.jsonl').read().strip().splitlines()[-1])
print('$f', round(d.get('value',0),3), (d.get('e2e') or {}).get('value'), d.get('parity'), d.get('config',{}).get('workload'), (d.get('clocks') or {}).get('reasons'), (d.get('roofline') or {}).get('frac'), (d.get('roofline_ntt') or {}).get('frac'))"; done
python tools/pipes.py > gpurun_out/r02_pipes.json 2>&1
bash tools/gpu_profile.sh 64 "ks_inner_mix moddown_pair ntt_inverse_kernel" > gpurun_out/prof64.log 2>&1; echo "profile rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:ntt_" -c 2 -o /tmp/prof_ntt python tools/ntt_launch.py > gpurun_out/ncu_ntt.log 2>&1; echo "ncu ntt rc=$?"
ncu -i /tmp/prof_ntt.ncu-rep --page raw --csv > gpurun_out/full_ntt.csv
ncu -i /tmp/prof_ntt.ncu-rep --page source --csv > gpurun_out/source_ntt.csv 2>/dev/null
head -14 gpurun_out/prof64.log
