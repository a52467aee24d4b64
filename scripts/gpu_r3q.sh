# config-4 sweep re-measured with the non-blocking cli.measure, plus per-step launch efficiency
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/sweep
timeout 900 python scripts/probe_steps.py > gpurun_out/sweep/probe_steps.log 2>&1
bash scripts/sweep_config4.sh
