TRACES="trace_b1" bash scripts/trace_run.sh; cat gpurun_out/trace_b1.log
