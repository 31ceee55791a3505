TRACES="trace_dq" bash scripts/trace_run.sh; cat gpurun_out/trace_dq.log
