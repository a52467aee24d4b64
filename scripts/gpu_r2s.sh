# CUDA-graph replay of the TokenRing runner: parity (single rank + shared-
# device multi-process on every transport), and host enqueue vs device time
# of 8-process shared-device runs with and without the graph.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_execute.py tests/test_gpu_ring_ipc.py -q -x -k "graph" > $O/pytest_graph.log 2>&1; echo "rc=$?" >> $O/pytest_graph.log
tail -4 $O/pytest_graph.log
for g in --no-graph --graph; do
 for S in 32768 131072; do
  TR_BENCH_SHARED_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \
    --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 8 --steps 5 --warmup 3 --seq $S \
    --transport fused --no-cpu-baseline --no-e2e $g > $O/bench_shared_${S}_p8$g.json 2> $O/bench_shared_${S}_p8$g.err
  python -c "import json; d=json.load(open('$O/bench_shared_${S}_p8$g.json')); print('S=$S P=8 $g: ms/step', round(d['ms_per_step'],3), 'host enqueue ms/step', round(d['host_enqueue_ms_per_step'],3), 'graph', d['cuda_graph'], 'launches', d['gpu_launches'])" || tail -5 $O/bench_shared_${S}_p8$g.err
 done
done
