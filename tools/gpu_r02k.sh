bash tools/gpu_quick.sh r02k "window or c1_all or stream or bit or c0_T10 or single_instance_754 or context or detect" "C1|context"
bash tools/gpu_sanitize.sh r02k_san
cat gpurun_out/r02k_san_summary.txt
