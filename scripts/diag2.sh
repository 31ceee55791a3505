TRACES="trace_fwd" bash scripts/trace_run.sh; cat gpurun_out/trace_fwd.log
