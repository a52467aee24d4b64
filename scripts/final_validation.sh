set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
TAG=${TAG:-r01h} bash scripts/profile.sh > gpurun_out/f_profile.log 2>&1
tail -2 gpurun_out/f_pytest_gpu.log; tail -1 gpurun_out/f_smoke.log; cat gpurun_out/f_bench.json
