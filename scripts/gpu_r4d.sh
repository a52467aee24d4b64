# Stream-order semantics around programmatic dependent launches.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04d; mkdir -p $O
timeout 300 python scripts/probe_pdl_order.py > $O/probe_pdl_order.log 2>&1; echo "rc=$?" >> $O/probe_pdl_order.log
cat $O/probe_pdl_order.log
