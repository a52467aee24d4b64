set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02o; mkdir -p $O
V=paper_2412_20501_b200/_variants
TOKENRING_LIB=$V/lib_skip.so timeout 90 python scripts/ab_parity.py > $O/parity.log 2>&1; cat $O/parity.log
for l in base skip; do
  if [ $l = base ]; then L=paper_2412_20501_b200/libtokenring.so; else L=$V/lib_$l.so; fi
  echo "== $l" >> $O/probe.log
  TOKENRING_LIB=$L timeout 600 python scripts/probe_steps.py 32768 131072 >> $O/probe.log 2>&1
done
cat $O/probe.log
