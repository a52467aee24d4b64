# compute-sanitizer over every product kernel (scripts/sanitize_small.py) and a
# 2-process fused TokenRing forward sharing cuda:0 (IPC peer stores, flags).
mkdir -p gpurun_out/sanitize
S=compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $S --tool $tool --print-limit 50 python scripts/sanitize_small.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/summary.txt
  tail -3 gpurun_out/sanitize/$tool.log >> gpurun_out/sanitize/summary.txt
done
for tool in memcheck synccheck; do
  TR_BENCH_SHARED_DEVICE=1 timeout 900 $S --tool $tool --target-processes all --print-limit 50 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 1 --warmup 1 --seq 4096 --heads 2 --transport fused --no-cpu-baseline --no-e2e \
    > gpurun_out/sanitize/fused2_$tool.log 2>&1
  echo "fused2 $tool rc=$?" >> gpurun_out/sanitize/summary.txt
  grep -E "ERROR SUMMARY|Error|error" gpurun_out/sanitize/fused2_$tool.log | tail -4 >> gpurun_out/sanitize/summary.txt
done
cat gpurun_out/sanitize/summary.txt
