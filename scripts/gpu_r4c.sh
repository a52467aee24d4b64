# Programmatic dependent launch between one rank's step launches: probe + kernel tests.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > $O/pytest_kernels.log 2>&1; echo "pytest rc=$?" >> $O/pytest_kernels.log
tail -2 $O/pytest_kernels.log
timeout 900 python scripts/probe_pdl.py 32768 131072 > $O/probe_pdl.log 2>&1; echo "probe rc=$?" >> $O/probe_pdl.log
cat $O/probe_pdl.log
