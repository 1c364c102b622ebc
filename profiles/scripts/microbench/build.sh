# Builds the round-2 generation-kernel experiments (profiles/r02_microbench/README.md)
# into profiles/scripts/microbench/_bin (git-ignored). Run from the repo root.
set -e
D=profiles/scripts/microbench
mkdir -p $D/_bin
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17"
$NV -o $D/_bin/mb_base $D/mb_gen.cu                                   # R=13, VW=2 (the product shape)
for k in 1 2 4 7; do $NV -DVMT_SHR_FMA=$k -o $D/_bin/mb_shr$k $D/mb_gen.cu; done
$NV -DMB_VW=1 -o $D/_bin/mb_vw1 $D/mb_gen.cu
$NV -DMB_VW=2 -DVMT_GEN_MINB=2 -o $D/_bin/mb_2cta $D/mb_gen.cu       # run with args: 20 296
$NV -DMB_R=4 -DMB_VW=4 -DVMT_GEN_MINB=1 -o $D/_bin/mb_r4v4 $D/mb_gen.cu
$NV -DMB_TMA=true -o $D/_bin/mb_tma208 $D/mb_gen.cu
# (VMT_PAIR128, the shuffle-paired 128-bit stores of pair128.log, was removed from the kernel after it measured slower)
$NV -DNC=256 -DCV=2 -o $D/_bin/ws_256 $D/ws_gen.cu
$NV -o $D/_bin/probe_st $D/probe_st.cu
$NV -o $D/_bin/pipes $D/pipes.cu                                      # pipe rates (pipes.log)
$NV -DSV=4 -o $D/_bin/split_v4 $D/split_gen.cu                        # runs of 6/7, 4 lanes per thread
$NV -DSV=2 -o $D/_bin/split_v2 $D/split_gen.cu                        # runs of 6/7, 512 threads
$NV -o $D/_bin/inplace $D/inplace_gen.cu                              # in-place ring, static slots
$NV -o $D/_bin/probe_power $D/probe_power.cu                          # store paths: rate + power (power.sh)
$NV -DSTAGE=1 -o $D/_bin/inplace_tma $D/inplace_gen.cu                  # + TMA bulk stores of double-buffered windows
$NV -o $D/_bin/qmajor $D/qmajor_gen.cu                                # lane-pair-major ring, 128-bit ring accesses
