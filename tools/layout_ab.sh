# Same-box A/B of the stage-1 layouts of the in-tree library: bit-identity
# hashes, then warm timings (prof_minors prints a cold and a warm call).
# usage (under gpurun): LAYOUTS="wide wide8" N=4096 R=441 bash tools/layout_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lay in ${LAYOUTS:-wide wide8}; do
  for sz in "1031 40" "4096 20"; do
    echo "== hash $lay $sz" >> gpurun_out/layout_ab.log
    EIGENID_STAGE1_LAYOUT=$lay timeout 300 python tools/spectra_hash.py $sz >> gpurun_out/layout_ab.log 2>&1
  done
done
for rep in $(seq ${REPS:-1}); do
  for lay in ${LAYOUTS:-wide wide8}; do
    echo "== time $lay" >> gpurun_out/layout_ab.log
    EIGENID_STAGE1_LAYOUT=$lay EIGENID_PROFILE=1 timeout 300 python tools/prof_minors.py ${N:-4096} ${R:-441} >> gpurun_out/layout_ab.log 2>&1
  done
done
