# A/B of library builds: per build, the CTA-0 trace (cycles per kv tile,
# clock-independent) and the power-capped sustained throughput (6 s loops,
# 32K causal and 8K x 16K full), two interleaved rounds.
#   bash scripts/ab_libs.sh OUT name1=lib1.so name2=lib2.so ...
# a name starting with "trace" is only traced.
out=$1; shift
mkdir -p $(dirname $out)
for round in 1 2; do
 for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  case $name in
   trace*) echo "== $name round $round" >> $out
           TOKENRING_LIB=$lib timeout 300 python scripts/trace_pair2.py 2>&1 | head -6 >> $out ;;
   *) echo "== $name round $round" >> $out
      TOKENRING_LIB=$lib timeout 120 python scripts/power_probe.py attn-causal 6 >> $out 2>&1
      TOKENRING_LIB=$lib timeout 120 python scripts/power_probe.py attn-full 6 >> $out 2>&1 ;;
  esac
 done
done
