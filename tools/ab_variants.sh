# A/B timing of compile-time variants of the device library (development aid).
# usage (under gpurun):
#   VARIANTS='base: ;wide:-DEIGENID_STAGE1_WIDE=1' N=4096 R=591 REPS=2 bash tools/ab_variants.sh
# A variant spec may end in '|<dir>': sources present in <dir> replace the
# in-tree ones of the same name (e.g. an older kernel file for a same-box A/B).
# LAYOUT=wide|narrow|wide8 picks the stage-1 layout (default: by n).
# Each variant is built into /tmp/ab_<name> and timed with tools/prof_minors.py
# (lambda(A) + R minor spectra); per-stage device times go to gpurun_out/ab.log.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${N:-4096}; R=${R:-591}; REPS=${REPS:-2}
build() {  # $1 = out dir, $2 = extra nvcc flags, $3 = override dir (optional)
  mkdir -p $1
  for f in paper_2002_04989_b200/csrc/*.cu; do
    src=$f
    [ -n "$3" ] && [ -f "$3/$(basename $f)" ] && src=$3/$(basename $f)
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 $2 -I paper_2002_04989_b200/csrc -Xcompiler -fPIC -c $src -o $1/$(basename $f).o &
  done; wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $1/libeigenid_b200.so $1/*.o
}
names=()
IFS=';' read -ra specs <<< "$VARIANTS"
for spec in "${specs[@]}"; do
  name=${spec%%:*}; rest=${spec#*:}
  flags=${rest%%|*}; over=""
  [ "$rest" != "$flags" ] && over=${rest#*|}
  names+=("$name")
  build /tmp/ab_$name "$flags" "$over" &
done
wait
for rep in $(seq $REPS); do
  for name in "${names[@]}"; do
    echo "== $name" >> gpurun_out/ab.log
    EIGENID_STAGE1_LAYOUT=${LAYOUT:-} EIGENID_LIB=/tmp/ab_$name/libeigenid_b200.so EIGENID_PROFILE=1 timeout 300 \
      python tools/prof_minors.py $N $R >> gpurun_out/ab.log 2>&1
  done
done
