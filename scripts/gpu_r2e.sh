mkdir -p gpurun_out/r02e
# parity of the split kernel: run the kernel + execute tests with it as the product library
cp paper_2412_20501_b200/libtokenring.so /tmp/lib_product.so
cp paper_2412_20501_b200/_variants/lib_split.so paper_2412_20501_b200/libtokenring.so
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_execute.py -x -q -k "not single_cta" > gpurun_out/r02e/pytest_split.log 2>&1
tail -3 gpurun_out/r02e/pytest_split.log
cp /tmp/lib_product.so paper_2412_20501_b200/libtokenring.so
TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_split.so timeout 300 python scripts/trace_pair2s.py > gpurun_out/r02e/trace_split.log 2>&1
bash scripts/ab_libs.sh gpurun_out/r02e/ab_split.log base=paper_2412_20501_b200/libtokenring.so split=paper_2412_20501_b200/_variants/lib_split.so
