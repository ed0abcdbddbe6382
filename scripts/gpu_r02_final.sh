# usage: bash scripts/gpu_r02_final.sh   (under gpurun --gpus 4): evidence after the last kernel change of round 2 --
# full pytest -m gpu, bench lines N = 1, 2, 4 x every config (+ reference arms), bf16 wire dyn vs stride, one-clock
# breakdown at NiN p = 2, 4
O=gpurun_out/r02_final; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu_4gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
for c in nin googlenet alexnet vgg19; do
  timeout 600 python bench.py --config $c > $O/bench_n1_$c.json 2> $O/bench_n1_$c.err
done
for N in 2 4; do for c in nin googlenet alexnet vgg19; do
  timeout 900 $TR --nproc-per-node $N --master-port 29611 bench.py --gpus $N --config $c > $O/bench_n${N}_$c.json 2> $O/bench_n${N}_$c.err
done; done
timeout 600 python bench.py --impl reference > $O/ref_n1_nin.json 2> $O/ref_n1_nin.err
for N in 2 4; do timeout 600 $TR --nproc-per-node $N --master-port 29612 bench.py --impl reference --gpus $N > $O/ref_n${N}_nin.json 2> $O/ref_n${N}_nin.err; done
for N in 2 4; do for rep in 1 2; do for M in dyn stride; do
  FC_FLAT_MAP=$M timeout 600 $TR --nproc-per-node $N --master-port 29613 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "N=$N $M rep$rep $(python -c "import json;d=json.load(open('$O/b.json'));b=d['baselines_ms_per_step'];print('flat', d['ms_per_step'], 'bf16', b['flat_bf16_wire_ms'], d['parity']['executors']['flat_bf16_wire'])")" >> $O/bf16_map.txt
done; done; done
for N in 2 4; do timeout 300 $TR --nproc-per-node $N --master-port 29614 scripts/gap_coll.py --size 7600000 --dump 2>/dev/null | grep -v NCCL > $O/gap_n$N.jsonl; done
echo done
