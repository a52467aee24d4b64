# Trigger only when asked (TR_LAUNCH_RELEASE_NEXT): A/B of the plain launch vs the
# pre-PDL build, chain probe, order probe, runner + cli GPU tests.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04i; mkdir -p $O
bash scripts/ab_libs.sh $O/cond_trigger_ab.log pre=scripts/ab/libtokenring_prepdl.so cond=scripts/ab/libtokenring_cond.so
bash scripts/ab_libs.sh $O/cond_trigger_ab2.log cond=scripts/ab/libtokenring_cond.so pre=scripts/ab/libtokenring_prepdl.so
grep -h "==\|attn" $O/cond_trigger_ab.log $O/cond_trigger_ab2.log | awk '{print $1,$2,$3,$4}'
timeout 900 python scripts/probe_pdl.py 32768 131072 > $O/probe_pdl.log 2>&1; cat $O/probe_pdl.log
timeout 300 python scripts/probe_pdl_order.py > $O/probe_pdl_order.log 2>&1; tail -3 $O/probe_pdl_order.log
timeout 1200 python -m pytest tests/test_gpu_ring_ipc.py tests/test_cli.py tests/test_gpu_kernels.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
