# Runner with overlapped (programmatic dependent) step launches: the whole GPU suite.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04e; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ring_ipc.py -x -q -m gpu -k overlapped > $O/pytest_overlap.log 2>&1; echo "pytest rc=$?" >> $O/pytest_overlap.log
tail -3 $O/pytest_overlap.log
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
