set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02m; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in rs rs48 rs_poly4; do TOKENRING_LIB=$V/lib_$l.so timeout 90 python scripts/ab_parity.py >> $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log; done
cat $O/parity.log
if grep -q "lib_rs.so: PASS" $O/parity.log; then
for l in trace_pair2 trace_rs; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py >> $O/traces.log 2>&1
done
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so rs=$V/lib_rs.so rspoly4=$V/lib_rs_poly4.so rs48=$V/lib_rs48.so
fi
grep -E "==|MMA period|half|exp c0" $O/traces.log; grep -E "^==|TFLOP" $O/ab.log
