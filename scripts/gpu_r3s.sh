# shared-device rehearsal of the multi-rank bench with the e2e leg (edge
# pieces, per-size runners over IPC) at 2 and 4 ranks on one GPU
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3s; mkdir -p $O
for n in 2 4; do
  TR_BENCH_SHARED_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 3 --warmup 3 --seq 32768 \
    --no-cpu-baseline > $O/bench_shared_$n.json 2> $O/bench_shared_$n.err
  echo "n=$n rc=$?"; tail -c 400 $O/bench_shared_$n.err
  python -c "
import json;d=json.loads(open('$O/bench_shared_$n.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], json.dumps(d.get('e2e'))[:260], d.get('cuda_graph'))"
done
