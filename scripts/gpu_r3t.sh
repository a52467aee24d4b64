# S row loaded from TMEM as 2 x64 or 1 x128 loads instead of 4 x32
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3t; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in sl64 sl128; do TOKENRING_LIB=$V/lib_$l.so timeout 90 python scripts/ab_parity.py 2>&1 | tail -1; done > $O/parity.log; cat $O/parity.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so sl64=$V/lib_sl64.so sl128=$V/lib_sl128.so
grep -E "^==|TFLOP" $O/ab.log
