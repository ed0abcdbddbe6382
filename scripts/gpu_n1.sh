set -x
B="python bench.py --steps 5 --warmup 2 --no-baselines --no-cpu-baseline"
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
for u in 1 2 4 8; do python bench.py --steps 200 --warmup 20 --no-baselines --no-cpu-baseline --sgd-unroll $u > gpurun_out/bench_u$u.json 2>&1; done
python bench.py --config alexnet --no-cpu-baseline > gpurun_out/bench_alexnet.json 2>&1
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv $B > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgd_step -s 3 -c 1 -o gpurun_out/prof_sgd $B > gpurun_out/ncu2.log 2>&1
echo done
