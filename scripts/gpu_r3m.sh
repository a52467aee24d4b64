# does the trace build's CTA-0 period track the untraced sustained throughput?
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3m; mkdir -p $O
V=paper_2412_20501_b200/_variants
for round in 1 2; do
for spec in base=paper_2412_20501_b200/libtokenring.so tbase=$V/lib_trace_base.so ss=$V/lib_ss.so tss=$V/lib_trace_ss.so; do
  n=${spec%%=*}; l=${spec#*=}
  echo "== $n"; TOKENRING_LIB=$l timeout 120 python scripts/power_probe.py attn-full 4 2>&1 | grep TFLOP
done
done > $O/ab.log; cat $O/ab.log
