# 3-chunk P split (64/32/32) A/B against the product (2 chunks, 96/32)
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3k; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in n3 n3p4; do TOKENRING_LIB=$V/lib_$l.so timeout 90 python scripts/ab_parity.py 2>&1 | tail -1; done > $O/parity.log; cat $O/parity.log
for l in base n3; do echo "== trace $l"; TOKENRING_LIB=$V/lib_trace_$l.so timeout 300 python scripts/trace_pair2.py 2>&1 | grep -E "MMA period|half|exp c0|pub"; done > $O/trace.log; cat $O/trace.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so n3=$V/lib_n3.so n3p4=$V/lib_n3p4.so
grep -E "^==|TFLOP" $O/ab.log
