mkdir -p gpurun_out
python tools/sweep_trace.py build/libpf_swtrace.so case9241 8 > gpurun_out/sweep_trace.txt 2>&1
cat gpurun_out/sweep_trace.txt
