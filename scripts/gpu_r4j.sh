# Final validation of the round-2 product with overlapped step launches: GPU suite,
# smoke, N=1 bench, shared-device multi-rank bench rehearsal (fused, graph replay),
# compute-sanitizer memcheck/synccheck of a 2-process fused forward.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04j; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
cat $O/bench.json
for n in 4; do
  TR_BENCH_SHARED_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 3 --warmup 3 --seq 32768 \
    --no-cpu-baseline > $O/bench_shared_$n.json 2> $O/bench_shared_$n.err
  echo "shared n=$n rc=$?"; tail -c 300 $O/bench_shared_$n.err
done
for tool in memcheck synccheck; do
  TR_BENCH_SHARED_DEVICE=1 timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 1 --warmup 1 --seq 4096 --heads 2 --transport fused --no-cpu-baseline --no-e2e \
    > $O/fused2_$tool.log 2>&1
  echo "fused2 $tool rc=$?" >> $O/sanitize_summary.txt
  grep -E "ERROR SUMMARY|Error|error" $O/fused2_$tool.log | tail -4 >> $O/sanitize_summary.txt
done
cat $O/sanitize_summary.txt
