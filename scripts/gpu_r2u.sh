set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02u; mkdir -p $O
timeout 120 python scripts/ab_parity.py > $O/parity.log 2>&1; cat $O/parity.log
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_execute.py tests/test_gpu_ring_ipc.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
for l in nosplit split; do
  if [ $l = split ]; then L=paper_2412_20501_b200/libtokenring.so; else L=paper_2412_20501_b200/_variants/lib_nosplit.so; fi
  for S in 32768 65536; do echo "== $l S=$S" >> $O/step0.log; TOKENRING_LIB=$L timeout 300 python scripts/probe_step0.py $S 8 >> $O/step0.log 2>&1; done
done
cat $O/step0.log
