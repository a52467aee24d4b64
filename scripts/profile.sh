#!/bin/bash
# Profiling recipe (run under gpurun, one GPU).  Outputs land in gpurun_out/.
#   1. launch list of one bench invocation (per-launch device time; cold-cache,
#      serialised -- compare shares, not absolutes)
#   2. one `ncu --set full` capture of the attention kernel at the bench size
#   3. one `ncu --set full` capture of the lse-merge kernel
#   4. one `ncu --set full` capture of the n-way merge (fused transport's fold)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 \
  -o gpurun_out/attn_${TAG} -f \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/attn_ncu_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_vec8 -c 1 \
  -o gpurun_out/merge_${TAG} -f \
  python scripts/probe_merge.py > gpurun_out/merge_ncu_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_n_bf16 -c 1 \
  -o gpurun_out/merge_n_${TAG} -f \
  python scripts/probe_merge.py > gpurun_out/merge_n_ncu_${TAG}.log 2>&1
ls -la gpurun_out
