timeout 900 python tools/config5.py > gpurun_out/config5_sim8.log 2>&1; echo "rc $?"; tail -2 gpurun_out/config5_sim8.log
