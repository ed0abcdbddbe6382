# usage: bash scripts/gpu_r02_nvl.sh N  (under gpurun --gpus N): NVLink bytes of the fused FLAT call on a real world
# (single-pass ncu metric set, every rank profiled), then the > 2^31-element parity tests
N=${1:-2}
O=gpurun_out/r02_nvl; mkdir -p $O
M=nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum
for c in nin alexnet; do
timeout 300 ncu --target-processes all --metrics $M --clock-control none -k regex:flat_kernel -s 3 -c 1 --csv \
  --log-file $O/nvl_${c}_n$N.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29591 scripts/real_flat_run.py $c > $O/nvl_${c}_n$N.log 2>&1
echo "$c ncu exit $?" >> $O/nvl_${c}_n$N.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "beyond_2_31" > $O/pytest_big.log 2>&1; echo "exit $?" >> $O/pytest_big.log
echo done
