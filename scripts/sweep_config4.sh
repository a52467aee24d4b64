#!/bin/bash
# BASELINE config 4 on one B200: seq 32K -> 1M at P = 2, 4, 8, ring vs TokenRing
# (causal: contiguous causal ring vs zigzag TokenRing; non-causal: ring vs
# token-ring).  Compute measured (every rank's step launches, max over ranks),
# exchange modelled on the NVSwitch port model.  Outputs: gpurun_out/sweep/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sweep
for P in 2 4 8; do
  for mode in causal noncausal; do
    python - "$P" "$mode" <<'PY'
import json, sys
P, mode = int(sys.argv[1]), sys.argv[2]
c = json.load(open(f"configs/b200_sweep_{mode}.json"))
c["parallel"]["ranks"] = P
json.dump(c, open(f"gpurun_out/sweep/cfg_{mode}_p{P}.json", "w"))
PY
    if [ "$mode" = causal ]; then sch=ring,zigzag-token-ring; else sch=ring,token-ring; fi
    timeout 900 python -m paper_2412_20501_b200.cli compare --config gpurun_out/sweep/cfg_${mode}_p${P}.json \
      --schedules $sch --sweep seq_len=32768..1048576 > gpurun_out/sweep/compare_${mode}_p${P}.csv \
      2> gpurun_out/sweep/compare_${mode}_p${P}.err
    echo "P=$P $mode rc=$?"
  done
done
