cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name --format=csv
timeout 600 python /root/repo/tests/_gpu_quick.py 2>&1 | tee gpurun_out/quick.log
