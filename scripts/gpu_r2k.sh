set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02k; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in s_poly4 s_poly6 s_poly3 s_skew20 s_skew24; do TOKENRING_LIB=$V/lib_$l.so timeout 120 python scripts/ab_parity.py >> $O/parity.log 2>&1; done
for l in trace_s_poly4; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py >> $O/traces.log 2>&1
done
bash scripts/ab_libs.sh $O/ab.log m1swp=$V/lib_m1swp.so poly4=$V/lib_s_poly4.so poly6=$V/lib_s_poly6.so poly3=$V/lib_s_poly3.so skew20=$V/lib_s_skew20.so skew24=$V/lib_s_skew24.so
grep -E "PASS|FAIL" $O/parity.log; grep -E "==|MMA period|half|exp c0" $O/traces.log; grep -E "^==|TFLOP" $O/ab.log
