mkdir -p gpurun_out/r02c
TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_pair2.so timeout 300 python scripts/trace_pair2.py > gpurun_out/r02c/trace_pair2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02c/pytest_new.log 2>&1
bash scripts/sanitize.sh > gpurun_out/r02c/sanitize.log 2>&1
