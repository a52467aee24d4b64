# After the programmatic-dependent-launch change: bench N=1 (product kernel now
# triggers its dependents), launch list + ncu of the attention kernel, config-5
# profile with chained step launches.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04g; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
cat $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_r04g.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches_bench_r04g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 \
  -o $O/attn_r04g -f \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/attn_ncu_r04g.log 2>&1
timeout 900 python -m paper_2412_20501_b200.cli profile --config configs/b200_config5_1m_h64.json \
  --trace $O/trace_config5_p8.json --summary $O/summary_config5_p8.csv > $O/profile_config5.log 2>&1
cat $O/profile_config5.log
ls -la $O
