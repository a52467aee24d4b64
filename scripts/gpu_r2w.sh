# Round-2 validation of the committed product: GPU tests, smoke, bench (N=1),
# reference arm, launch list + ncu of attention and merges, cuDNN side by side.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02w; mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1700 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
cat $O/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
TAG=r02w bash scripts/profile.sh > $O/profile.log 2>&1
mv gpurun_out/launches_r02w.csv gpurun_out/*_r02w.ncu-rep gpurun_out/*_r02w*.log $O/ 2>/dev/null
timeout 600 python scripts/calib_cudnn.py 6 > $O/calib_cudnn.log 2>&1
cat $O/calib_cudnn.log
