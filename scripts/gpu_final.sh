# usage: bash scripts/gpu_final.sh  — full GPU test suite + driver-style benches at N=4,2,1 (all configs), on a 4-GPU box
set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_final.log
bash scripts/gpu_bench.sh 4 r5
bash scripts/gpu_bench.sh 2 r5
export CUDA_VISIBLE_DEVICES=0
bash scripts/gpu_bench.sh 1 r5
for c in googlenet alexnet vgg19; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-baselines > gpurun_out/bench_r5_n1_$c.json 2> gpurun_out/bench_r5_n1_$c.err; done
