# usage: bash scripts/gpu_shared_gpu_worlds.sh — real (CUDA-IPC) worlds with several ranks per GPU
# (gloo bootstrap): 2 on 1 GPU, 4 on 2, 4 on 4, 8 on 4, 6 on 2; every schedule + stress bit-exact
run() { # name nproc gpus
  FC_MP_GPUS=$3 FC_MP_SIZES=5,16391,300007 FC_MP_STRESS=40 FC_MP_TIMEOUT=30 FC_MP_TIMEOUT_TEST=0 timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $2 --master-port $4 tests/mp_worker.py > gpurun_out/sh_$1.log 2>&1
  echo "$1 nproc=$2 gpus=$3 rc=$? ok=$(grep -o 'MP_OK [0-9]' gpurun_out/sh_$1.log | wc -l)"; grep -h "FAILS" gpurun_out/sh_$1.log | cut -c1-200 | head -4
}
run a 2 1 29701
run b 4 2 29702
run c 4 4 29703
run d 8 4 29704
run e 6 2 29705
