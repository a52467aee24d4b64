set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02p; mkdir -p $O
V=paper_2412_20501_b200/_variants
for l in base noorder skip base; do
  if [ $l = base ]; then L=paper_2412_20501_b200/libtokenring.so; else L=$V/lib_$l.so; fi
  for S in 32768 131072; do
    echo "== $l S=$S" >> $O/probe.log
    TOKENRING_LIB=$L timeout 300 python scripts/probe_step0.py $S 8 >> $O/probe.log 2>&1
  done
done
cat $O/probe.log
