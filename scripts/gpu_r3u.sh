# MMA-issuer P waits and/or softmax S waits polled with test_wait instead of try_wait
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3u; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in mspin sspin bspin; do TOKENRING_LIB=$V/lib_$l.so timeout 90 python scripts/ab_parity.py 2>&1 | tail -1; done > $O/parity.log; cat $O/parity.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so mspin=$V/lib_mspin.so sspin=$V/lib_sspin.so bspin=$V/lib_bspin.so
grep -E "^==|TFLOP" $O/ab.log
