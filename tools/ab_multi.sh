# Several ab_variants.sh rounds in one gpurun call, one per stage-1 layout.
# usage: ROUNDS="wide|<variants>#wide8|<variants>" bash tools/ab_multi.sh
cd $GRAFT_REPO_ROOT
IFS='#' read -ra rounds <<< "$ROUNDS"
for r in "${rounds[@]}"; do
  lay=${r%%|*}; vars=${r#*|}
  echo "#### layout $lay" >> gpurun_out/ab.log
  LAYOUT=$lay VARIANTS="$vars" N=${N:-4096} R=${R:-441} REPS=${REPS:-1} bash tools/ab_variants.sh
done
