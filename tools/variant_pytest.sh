# Runs the GPU parity suite against a variant build of the device library.
# usage: VARIANT="-DFOO=1" bash tools/variant_pytest.sh [pytest args]
set -e
cd $GRAFT_REPO_ROOT
out=/tmp/var_$(echo "$VARIANT" | md5sum | cut -c1-8)
mkdir -p $out
for f in paper_2002_04989_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 $VARIANT -Xcompiler -fPIC -c $f -o $out/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libeigenid_b200.so $out/*.o
EIGENID_LIB=$out/libeigenid_b200.so python -m pytest tests -m gpu "$@"
