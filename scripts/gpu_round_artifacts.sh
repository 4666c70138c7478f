#!/bin/bash
# Round artifacts on one GPU: headline bench (both arms), the other §8 workloads, the ncu launch
# list of the bench command, ncu captures of the network, guard, setup and fused per-pixel kernels,
# and of the trainer's GEMM.  Summarised into profiles/ by scripts/summarize_profiles.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-300
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
timeout 600 python scripts/bench_configs.py --out gpurun_out/configs.jsonl > /dev/null 2> gpurun_out/configs.err; wc -l gpurun_out/configs.jsonl
# launch list of the same command (cold-cache, serialised per-launch times)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches rc=$?
# network kernel as benchmarked (cluster-multicast pair): counters only -- the full set's source-level
# instrumentation hangs the multicast cluster kernel; the full set with source is taken on the
# single-CTA variant (same MMA / epilogue / encoder code, no multicast)
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic,launch__cluster_dim_x,sm__throughput.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -k regex:nedf_mlp_tc_kernel -s 2 -c 1 \
  -o gpurun_out/tc_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tc.log 2>&1; echo tc rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:nedf_mlp_tc_kernel -s 2 -c 1 \
  -o gpurun_out/tc_single_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --tc-kernel single > gpurun_out/ncu_tc_single.log 2>&1; echo tc single rc=$?
for k in guard_tc_kernel setup_kernel resolve_shade_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/${k}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$k.log 2>&1; echo $k rc=$?
done
# the trainer: launch list of 3 paper-profile iterations and one forward-body GEMM
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/train_launches.csv \
  python scripts/train_profile.py 3 > gpurun_out/ncu_train.log 2>&1; echo train launches rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3 -s 105 -c 1 \
  -o gpurun_out/gemm_full python scripts/train_profile.py 2 > gpurun_out/ncu_gemm.log 2>&1; echo gemm rc=$?
