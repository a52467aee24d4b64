# persistent pair kernel (TR_P2_PERSIST): parity gate, the GPU suites run on it
# (box-local copy swapped in as the product library), then the sustained A/B
# and the small-S step geometry
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3r; mkdir -p $O
V=paper_2412_20501_b200/_variants
TOKENRING_LIB=$V/lib_persist.so timeout 120 python scripts/ab_parity.py > $O/parity.log 2>&1; tail -3 $O/parity.log
grep -q PASS $O/parity.log || exit 3
cp paper_2412_20501_b200/libtokenring.so /tmp/lib_product.so
cp $V/lib_persist.so paper_2412_20501_b200/libtokenring.so
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_execute.py tests/test_gpu_fullsize.py tests/test_gpu_ring_ipc.py -q -x > $O/pytest_persist.log 2>&1; tail -3 $O/pytest_persist.log
cp /tmp/lib_product.so paper_2412_20501_b200/libtokenring.so
for l in base=paper_2412_20501_b200/libtokenring.so persist=$V/lib_persist.so; do
  n=${l%%=*}; f=${l#*=}
  echo "== $n"; TOKENRING_LIB=$f timeout 300 python scripts/probe_step0.py 32768 8 2>&1 | head -9
done > $O/step0.log 2>&1; cat $O/step0.log
bash scripts/ab_libs.sh $O/ab.log base=paper_2412_20501_b200/libtokenring.so persist=$V/lib_persist.so
grep -E "^==|TFLOP" $O/ab.log
