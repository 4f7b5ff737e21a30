cd $GRAFT_REPO_ROOT
timeout 600 python tools/gpu_quick.py 2>&1 | tee gpurun_out/quick.log
EIGENID_PROFILE=1 timeout 900 python tools/prof_pipeline.py ${1:-1024} ${2:-2} 2>&1 | tee gpurun_out/time.log
