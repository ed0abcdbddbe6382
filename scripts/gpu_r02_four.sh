# usage: bash scripts/gpu_r02_four.sh   (under gpurun --gpus 4): full pytest -m gpu, exit-protocol decomposition,
# FLAT mapping A/B at p=4, bench lines N=1/2/4 (GoogLeNet with every executor, PS and NCCL baselines), f3 overlap
mkdir -p gpurun_out/r02_four
O=gpurun_out/r02_four
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu_4gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_4gpu.log
timeout 300 ./scripts/gap_bench > $O/gap_bench.txt 2>&1
for rep in 1 2; do for M in balanced dyn; do
  FC_FLAT_MAP=$M timeout 300 $TR --nproc-per-node 4 --master-port 29561 scripts/gap_coll.py --size 7600000 --dump 2>/dev/null | grep '"fused"' | sed "s/^/$M rep$rep /" >> $O/flat_map_p4.txt
  FC_FLAT_MAP=$M timeout 600 $TR --nproc-per-node 4 --master-port 29562 bench.py --gpus 4 --steps 200 --warmup 20 --no-baselines --no-cpu-baseline > $O/map_bench_${M}.json 2>/dev/null
  echo "$M rep$rep bench $(python -c "import json;d=json.load(open('$O/map_bench_${M}.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'])")" >> $O/flat_map_p4.txt
done; done
for N in 4 2; do for c in nin googlenet alexnet vgg19; do
  timeout 900 $TR --nproc-per-node $N --master-port 29563 bench.py --gpus $N --config $c > $O/bench_n${N}_$c.json 2> $O/bench_n${N}_$c.err
done; done
timeout 600 python bench.py > $O/bench_n1_nin.json 2> $O/bench_n1_nin.err
timeout 600 python bench.py --impl reference > $O/ref_n1_nin.json 2> $O/ref_n1_nin.err
timeout 600 $TR --nproc-per-node 4 --master-port 29564 bench.py --impl reference --gpus 4 > $O/ref_n4_nin.json 2> $O/ref_n4_nin.err
for N in 4 2; do
  timeout 900 $TR --nproc-per-node $N --master-port 29565 examples/nin_dp_torchrun.py --steps 20 > $O/nin_dp_n$N.json 2> $O/nin_dp_n$N.err
done
echo done
