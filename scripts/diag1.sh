mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2204_07143_b200/csrc -I include -o /tmp/tmem_bw scripts/microbench_tmem_bw.cu && timeout 120 /tmp/tmem_bw > gpurun_out/tmem_bw.txt 2>&1
TRACES="trace_b1" bash scripts/trace_run.sh > /dev/null 2>&1
ls gpurun_out
