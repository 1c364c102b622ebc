#!/bin/bash
# Round-2 captures (run on the B200 box from the repo root; each command first
# runs without ncu and must exit 0):
#   gen     ncu --set full of the store-mode generation kernel (in-place ring)
#   steady  ncu app-range replay of ONE bench step (2^34 words, L=32): the
#           generation kernel with the next step's tcgen05 positioning GEMM
#           running beside it, kernels concurrent as in the bench
#   c1      launch list of config 1's fills
#   jump    ncu --set full of config 5's jump kernel
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
set -x
python profiles/scripts/prof_target.py gen || exit 1
ncu --set full --clock-control none --import-source on -k regex:vmt_gen_kernel --launch-skip 2 -c 1 \
    -o $OUT/r02_prof_gen -f python profiles/scripts/prof_target.py gen > $OUT/r02_ncu_gen.log 2>&1
python profiles/scripts/prof_target.py steady || exit 1
M=gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__cycles_elapsed.avg.per_second
ncu --replay-mode app-range --clock-control none --metrics $M --csv \
    --log-file $OUT/r02_steady_range.csv python profiles/scripts/prof_target.py steady > $OUT/r02_ncu_steady.log 2>&1
# the bench's own 2^34-word store launch (roofline.traffic measured on it, not scaled)
python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu-baseline > $OUT/r02_bench_small.json || exit 1
ncu --set full --clock-control none -k regex:vmt_gen_kernel --launch-skip 1 -c 1 -o $OUT/r02_prof_gen_bench -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu-baseline > $OUT/r02_ncu_gen_bench.log 2>&1
python profiles/scripts/prof_target.py c1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_launches_c1.csv \
    python profiles/scripts/prof_target.py c1 > $OUT/r02_ncu_c1.log 2>&1
python profiles/scripts/prof_target.py c5 || exit 1
ls -la $OUT
ncu --set full --clock-control none --import-source on -k regex:vmt_jump_kernel --launch-skip 1 -c 2 \
    -o $OUT/r02_prof_c5 -f python profiles/scripts/prof_target.py c5 > $OUT/r02_ncu_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_launches_c5.csv \
    python profiles/scripts/prof_target.py c5 > $OUT/r02_ncu_c5l.log 2>&1
