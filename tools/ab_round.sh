# One gpurun call for a kernel change: bit-identity hash (old vs new build),
# A/B timing, then the per-phase clock64 split of the new build.
# usage (under gpurun): OLD=build/ab_old FLAGS="..." bash tools/ab_round.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="old: |${OLD:-build/ab_old};new:${FLAGS:- }" N=${N:-4096} R=${R:-441} REPS=${REPS:-2} bash tools/ab_variants.sh
for name in old new; do
  for sz in "1031 40" "4096 20"; do
    echo "== hash $name $sz" >> gpurun_out/ab.log
    EIGENID_LIB=/tmp/ab_$name/libeigenid_b200.so timeout 300 python tools/spectra_hash.py $sz >> gpurun_out/ab.log 2>&1
  done
done
EIGENID_STAGE1_LAYOUT=wide EIGENID_LIB=/tmp/ab_new/libeigenid_b200.so timeout 300 python tools/spectra_hash.py 1031 40 >> gpurun_out/ab.log 2>&1
echo "== hash old wide 1031" >> gpurun_out/ab.log; EIGENID_STAGE1_LAYOUT=wide EIGENID_LIB=/tmp/ab_old/libeigenid_b200.so timeout 300 python tools/spectra_hash.py 1031 40 >> gpurun_out/ab.log 2>&1
if [ -n "$PHASES" ]; then N=4096 R=146 SLOTS=148 bash tools/phase_timing.sh > gpurun_out/phases.log 2>&1; fi
