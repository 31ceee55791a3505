cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
NA2D_PARITY_LOG=gpurun_out/r02_parity_errors_v8.jsonl timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_v8.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_v8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v8.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_v8.log
tail -2 gpurun_out/pytest_gpu_v8.log; tail -1 gpurun_out/smoke_v8.log
timeout 600 python bench.py > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err; echo "bench exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_v8.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu_bench_v8.log 2>&1
for k in na2d_fwd_tc na2d_bwd_dq na2d_bwd_dkdv; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 2 -c 1 -o gpurun_out/full_v8_$k -f python scripts/prof_fwd.py cfg2_nat_tiny_s1 4 --bwd > gpurun_out/ncu_v8_$k.log 2>&1
done
python scripts/ncu_summary.py gpurun_out/ncu_full_v8.md cfg2_nat_tiny_s1 gpurun_out/full_v8_*.ncu-rep
bash scripts/bench_configs.sh
: > gpurun_out/r02_f3.jsonl
for c in f3_d16_s1 f3_d64_s1; do python bench.py --config $c --steps 10 --warmup 3 --no-extras 2>/dev/null | tail -1 >> gpurun_out/r02_f3.jsonl; done
timeout 300 python scripts/simt_timing.py > gpurun_out/r02_simt_timing.txt 2>&1
