set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02i; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in mma1 mt1 mt1_pp mt1_pp2 mt1_tree; do TOKENRING_LIB=$V/lib_$l.so timeout 120 python scripts/ab_parity.py >> $O/parity.log 2>&1; done
for l in trace_pair2 trace_mt1; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py >> $O/traces.log 2>&1
done
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so mma1=$V/lib_mma1.so mt1=$V/lib_mt1.so mt1pp=$V/lib_mt1_pp.so mt1pp2=$V/lib_mt1_pp2.so mt1tree=$V/lib_mt1_tree.so
grep -E "PASS|FAIL" $O/parity.log; head -14 $O/traces.log; grep -A12 "== trace_mt1" $O/traces.log; grep -E "^==|TFLOP" $O/ab.log
