set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --batch 8 --steps 1 --warmup 3 --no-extras > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'ks_inner|moddown|ntt_inverse|ntt_forward' -s 40 -c 4 -o gpurun_out/prof python bench.py --batch 8 --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
