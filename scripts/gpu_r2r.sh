set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02r; mkdir -p $O
timeout 900 python scripts/probe_steps.py 32768 65536 131072 > $O/probe_steps.log 2>&1
cat $O/probe_steps.log
for n in 8; do
  TR_BENCH_SHARED_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n --steps 5 --warmup 3 --seq 32768 \
    --transport fused --no-cpu-baseline --no-e2e > $O/bench_shared_32k_p$n.json 2> $O/bench_shared_32k_p$n.err
  python -c "import json; d=json.load(open('$O/bench_shared_32k_p$n.json')); print('32K P=$n shared: ms/step', d['ms_per_step'], 'host enqueue ms/step', d['host_enqueue_ms_per_step'])"
done
