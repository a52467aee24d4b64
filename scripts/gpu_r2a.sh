set -x
mkdir -p gpurun_out/r02a
python -m pytest tests/test_gpu_ring_ipc.py tests/test_gpu_multidevice.py -q -x -k "ringattn or multidevice or distinct" 2>&1 | tail -15 > gpurun_out/r02a/pytest_ring.log
for sch in ring token-ring; do
 for n in 2 4; do
  TR_BENCH_SHARED_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $n --steps 3 --warmup 3 --seq 32768 --transport fused --schedule $sch --no-cpu-baseline --no-e2e > gpurun_out/r02a/bench_shared_${sch}_${n}.json 2> gpurun_out/r02a/bench_shared_${sch}_${n}.err
 done
done
TR_BENCH_SHARED_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 3 --seq 32768 --transport ipc --schedule ring --non-causal --no-cpu-baseline > gpurun_out/r02a/bench_shared_ring_nc_ipc_2.json 2> gpurun_out/r02a/bench_shared_ring_nc_ipc_2.err
