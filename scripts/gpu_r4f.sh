# Config-4 sweep (ring vs TokenRing, 32K -> 1M, P = 2, 4, 8) with each rank's
# chained step launches (programmatic dependent launches) beside the
# step-synchronous totals; config-3 chained profile.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04f; mkdir -p $O
timeout 300 python -m paper_2412_20501_b200.cli profile --config configs/b200_tokenring_128k.json \
  --trace $O/trace_128k_p8.json --summary $O/summary_128k_p8.csv > $O/profile_config3.log 2>&1
cat $O/profile_config3.log
bash scripts/sweep_config4.sh > $O/sweep.log 2>&1
cp -r gpurun_out/sweep $O/
python scripts/sweep_summary.py $O/sweep > $O/summary.md
cat $O/summary.md
