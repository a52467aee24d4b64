# Round 2 re-validation after the container re-creation: the committed product
# (GPU tests, smoke, bench, launch list + ncu), split-row A/B, cuDNN calibration,
# measured-lane traces of 4- and 8-process shared-device runs, sanitizers.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02f
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
cat $O/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
TAG=r02f bash scripts/profile.sh > $O/profile.log 2>&1
mv gpurun_out/launches_r02f.csv gpurun_out/*_r02f.ncu-rep gpurun_out/*_r02f*.log $O/ 2>/dev/null
# split-row softmax A/B (variant library vs product), clock-independent traces
bash scripts/ab_libs.sh $O/ab_split.log base=paper_2412_20501_b200/libtokenring.so split=paper_2412_20501_b200/_variants/lib_split.so
TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_pair2.so timeout 300 python scripts/trace_pair2.py > $O/trace_pair2.log 2>&1
TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_split.so timeout 300 python scripts/trace_pair2s.py > $O/trace_split.log 2>&1
timeout 600 python scripts/calib_cudnn.py 6 > $O/calib_cudnn.log 2>&1
# measured exchange lanes: 4- and 8-process shared-device runs, TokenRing and Ring
for n in 4 8; do
 for sch in token-ring ring; do
  TR_BENCH_SHARED_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 3 --warmup 3 \
    --transport fused --schedule $sch --no-cpu-baseline --trace-out $O/trace_${sch}_p$n \
    > $O/bench_shared_${sch}_p$n.json 2> $O/bench_shared_${sch}_p$n.err
 done
done
bash scripts/sanitize.sh > $O/sanitize.log 2>&1
mv gpurun_out/sanitize $O/ 2>/dev/null
ls -la $O
