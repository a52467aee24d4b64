# Re-validation after the container re-creation (rebuilt .so): GPU tests, smoke, bench.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04a; mkdir -p $O
nvidia-smi -L > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
cat $O/bench.json
