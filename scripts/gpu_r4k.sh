# The reference arm as the driver runs it (N=1), on the GPU box's host cores.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04k; mkdir -p $O
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?"
tail -c 600 $O/bench_ref.json
