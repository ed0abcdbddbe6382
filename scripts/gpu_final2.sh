# usage: bash scripts/gpu_final2.sh — end-of-round evidence on a 4-GPU box: full GPU test suite,
# driver-style benches (N = 4, 2, 1; every config; the reference arm), ncu launch list and
# --set full captures (1-GPU SGD at NiN and AlexNet size, FOREST and FLAT in a virtual world)
set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/f_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/f_pytest.log
bash scripts/gpu_bench.sh 4 f
bash scripts/gpu_bench.sh 2 f
export CUDA_VISIBLE_DEVICES=0
bash scripts/gpu_bench.sh 1 f
for c in googlenet alexnet vgg19; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-baselines > gpurun_out/bench_f_n1_$c.json 2> gpurun_out/bench_f_n1_$c.err
done
B="python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu-baseline"
$B > gpurun_out/f_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_n1.csv $B > gpurun_out/f_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgd_step -s 3 -c 1 -o gpurun_out/f_prof_sgd $B > gpurun_out/f_ncu2.log 2>&1
python scripts/sgd_run.py alexnet > gpurun_out/f_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sgd_step -s 2 -c 1 -o gpurun_out/f_prof_sgd_alexnet python scripts/sgd_run.py alexnet > gpurun_out/f_ncu3.log 2>&1
for s in flat forest; do
  python scripts/virtual_flat_run.py 4 $s > gpurun_out/f_plain_$s.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:${s}_kernel -s 2 -c 1 -o gpurun_out/f_prof_virtual_$s python scripts/virtual_flat_run.py 4 $s > gpurun_out/f_ncu_$s.log 2>&1
done
echo done
