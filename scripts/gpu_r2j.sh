set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02j; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in m1swp m1swp_pp2 m1_pp2 m1swp_tree; do TOKENRING_LIB=$V/lib_$l.so timeout 120 python scripts/ab_parity.py >> $O/parity.log 2>&1; done
for l in trace_m1 trace_m1swp; do
  echo "== $l" >> $O/traces.log
  TOKENRING_LIB=$V/lib_$l.so timeout 300 python scripts/trace_pair2.py >> $O/traces.log 2>&1
done
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so mma1=$V/lib_mma1.so m1swp=$V/lib_m1swp.so m1swppp2=$V/lib_m1swp_pp2.so m1pp2=$V/lib_m1_pp2.so m1swptree=$V/lib_m1swp_tree.so
grep -E "PASS|FAIL" $O/parity.log; grep -E "==|MMA period|half|exp c0" $O/traces.log; grep -E "^==|TFLOP" $O/ab.log
