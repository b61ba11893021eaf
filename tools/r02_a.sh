set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/trace_step.py --config c2 --graph > gpurun_out/r02_trace_c2_graph.txt 2>&1
python tools/trace_step.py --config c2 --graph --unfused > gpurun_out/r02_trace_c2_unfused_graph.txt 2>&1
python tools/trace_step.py --config c3 --graph > gpurun_out/r02_trace_c3_graph.txt 2>&1
tail -30 gpurun_out/r02_trace_c2_graph.txt
