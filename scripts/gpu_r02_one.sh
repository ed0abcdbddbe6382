# usage: bash scripts/gpu_r02_one.sh   (under gpurun, 1 GPU): the driver's round-end view -- full pytest -m gpu and
# smoke() on one GPU -- then bench N=1 (default line), the ncu launch list of the same command, ncu --set full of the
# 1-GPU SGD at NiN and VGG-19 size (traffic for roofline.traffic / steady_state.traffic) and of the FLAT kernel on a
# virtual 4-rank world (dynamic mapping) at NiN size
O=gpurun_out/r02_one; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu_1gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
B="python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu-baseline --no-steady"
$B > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_n1.csv $B > $O/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgd_step -s 3 -c 1 -o $O/prof_sgd_nin $B > $O/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgd_step -s 2 -c 1 -o $O/prof_sgd_vgg19 python scripts/sgd_run.py vgg19 > $O/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:flat_kernel -s 2 -c 1 -o $O/prof_flat_virtual_p4 python scripts/virtual_flat_run.py 4 flat > $O/ncu4.log 2>&1
echo done
