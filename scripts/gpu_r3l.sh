# split QK (S columns 64..127 of QK(j+1) issued ahead of P.V(j)) A/B against the product
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3l; mkdir -p $O
V=paper_2412_20501_b200/_variants
TOKENRING_LIB=$V/lib_ss.so timeout 90 python scripts/ab_parity.py > $O/parity.log 2>&1; tail -3 $O/parity.log
for l in base ss; do echo "== trace $l"; TOKENRING_LIB=$V/lib_trace_$l.so timeout 300 python scripts/trace_pair2.py 2>&1 | head -8; done > $O/trace.log 2>&1; cat $O/trace.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so ss=$V/lib_ss.so
grep -E "^==|TFLOP" $O/ab.log
