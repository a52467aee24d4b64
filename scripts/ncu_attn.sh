#!/bin/bash
# One ncu --set full capture of the attention kernel on config 2 (causal 32K).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-dev}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
  -o gpurun_out/attn_${TAG} -f python scripts/probe_attn.py --case 0 --iters 1 > gpurun_out/attn_${TAG}.log 2>&1
tail -3 gpurun_out/attn_${TAG}.log
