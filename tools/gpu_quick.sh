mkdir -p gpurun_out
timeout 600 python tools/motion_phases.py plaza > gpurun_out/motion.log 2>&1
