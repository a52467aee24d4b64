# A/B: product library with the griddepcontrol trigger (PDL) vs the build before it,
# sustained power-capped loops, two interleaved rounds.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r04h; mkdir -p $O
bash scripts/ab_libs.sh $O/pdl_trigger_ab.log pre=scripts/ab/libtokenring_prepdl.so pdl=scripts/ab/libtokenring_pdl.so
bash scripts/ab_libs.sh $O/pdl_trigger_ab2.log pdl=scripts/ab/libtokenring_pdl.so pre=scripts/ab/libtokenring_prepdl.so
cat $O/pdl_trigger_ab.log $O/pdl_trigger_ab2.log
