set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02v; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in late late_p4 late_p6; do TOKENRING_LIB=$V/lib_$l.so timeout 90 python scripts/ab_parity.py >> $O/parity.log 2>&1; done
grep -E "PASS|FAIL" $O/parity.log
for l in trace_pair2 trace_late; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py 2>&1 | head -12 >> $O/traces.log
done
grep -E "==|MMA period|half|exp c0" $O/traces.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so late=$V/lib_late.so latep4=$V/lib_late_p4.so latep6=$V/lib_late_p6.so
grep -E "^==|TFLOP" $O/ab.log
