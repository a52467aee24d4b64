set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02h; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in pp2 skew20_pp2; do TOKENRING_LIB=$V/lib_$l.so timeout 120 python scripts/ab_parity.py >> $O/parity.log 2>&1; done
for l in trace_pair2 trace_pp2 trace_skew20_pp2; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py 2>&1 | head -10 >> $O/traces.log
done
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so pp2=$V/lib_pp2.so skew20pp2=$V/lib_skew20_pp2.so
grep -E "PASS|FAIL" $O/parity.log; cat $O/traces.log; grep -E "^==|TFLOP" $O/ab.log
