set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3f; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in c96 c32; do TOKENRING_LIB=$V/lib_$l.so timeout 90 python scripts/ab_parity.py >> $O/parity.log 2>&1; done
grep -E "PASS|FAIL" $O/parity.log
for l in trace_pair2 trace_c96; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py 2>&1 | grep -E "MMA period|half|overlap" >> $O/traces.log
done
cat $O/traces.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so c96=$V/lib_c96.so c32=$V/lib_c32.so
grep -E "^==|TFLOP" $O/ab.log
