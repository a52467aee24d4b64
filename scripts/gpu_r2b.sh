mkdir -p gpurun_out/r02b
TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_pair2.so timeout 300 python scripts/trace_pair2.py > gpurun_out/r02b/trace_pair2_full.log 2>&1
TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_pair2.so timeout 300 python scripts/trace_pair2.py 8192 16384 32 128 >> gpurun_out/r02b/trace_pair2_full.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest_gpu.log 2>&1
tail -5 gpurun_out/r02b/pytest_gpu.log
