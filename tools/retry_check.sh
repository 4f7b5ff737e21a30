# Builds a variant that loses one mbarrier arrival (once) and checks that the
# bounded wait times out, the call is retried and the result is correct
# (development aid).  usage (under gpurun): bash tools/retry_check.sh
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/drop gpurun_out
for f in paper_2002_04989_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DEIGENID_EXP_DROP_ARRIVE -DEIGENID_WAIT_TIMEOUT_CYCLES=4000000000LL -I paper_2002_04989_b200/csrc -Xcompiler -fPIC -c $f -o /tmp/drop/$(basename $f).o &
done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/drop/libeigenid_b200.so /tmp/drop/*.o
EIGENID_LIB=/tmp/drop/libeigenid_b200.so EIGENID_PROFILE=0 FULL_REPS=2 timeout 300 python tools/full_run.py 2100 > gpurun_out/retry_check.log 2>&1
echo "rc=$?" >> gpurun_out/retry_check.log
