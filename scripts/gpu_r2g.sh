# A/B of the softmax-path variants suggested by the cuDNN calibration
# (tree max, heavier polynomial share in the first P chunk, ping-pong of the
# two halves): parity gate, CTA-0 traces, power-capped sustained throughput.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02g; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in tree tree_skew20 tree_skew40 tree_pp tree_skew20_pp tree_skew28; do
  TOKENRING_LIB=$V/lib_$l.so timeout 120 python scripts/ab_parity.py >> $O/parity.log 2>&1
done
for l in trace_pair2 trace_tree trace_tree_skew20 trace_tree_skew20_pp; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py 2>&1 | head -8 >> $O/traces.log
done
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so tree=$V/lib_tree.so \
  skew20=$V/lib_tree_skew20.so skew40=$V/lib_tree_skew40.so pp=$V/lib_tree_pp.so \
  skew20pp=$V/lib_tree_skew20_pp.so skew28=$V/lib_tree_skew28.so
grep -E "==|PASS|FAIL" $O/parity.log; grep -E "^==|TFLOP" $O/ab.log
