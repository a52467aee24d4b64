# Final round-2 validation of the product build:
# GPU tests, smoke, bench, launch list + ncu, cuDNN side by side.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02z; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
cat $O/bench.json
TAG=r02z bash scripts/profile.sh > $O/profile.log 2>&1
mv gpurun_out/launches_r02z.csv gpurun_out/*_r02z.ncu-rep gpurun_out/*_r02z*.log $O/ 2>/dev/null
timeout 600 python scripts/calib_cudnn.py 6 > $O/calib_cudnn.log 2>&1
cat $O/calib_cudnn.log
