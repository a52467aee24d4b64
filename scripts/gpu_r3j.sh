set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r3j; mkdir -p $O
V=paper_2412_20501_b200/_variants
timeout 90 python scripts/ab_parity.py > $O/parity.log 2>&1; tail -1 $O/parity.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_execute.py tests/test_gpu_fullsize.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
TOKENRING_LIB=$V/lib_trace_spec.so timeout 300 python scripts/trace_pair2.py 2>&1 | grep -E "MMA period|half|exp c0" > $O/trace.log; cat $O/trace.log
bash scripts/ab_libs.sh $O/ab.log prespec=$V/lib_prespec.so spec=paper_2412_20501_b200/libtokenring.so
grep -E "^==|TFLOP" $O/ab.log
