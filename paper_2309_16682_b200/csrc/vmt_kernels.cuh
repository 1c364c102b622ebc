// All sm_100a kernels of the VMT19937 build:
//   vmt_common.cuh  constants, parameters, twist/temper arithmetic, conversions
//   vmt_gen.cuh     vmt_gen_kernel: twist + temper + emit (the hot path)
//   vmt_jump.cuh    vmt_jump_kernel (polynomial jump-ahead), seeding, reduction
//   vmt_matrix.cuh  GF(2) jump matrices: basis states, effective layout, vec_mat_mul
//   vmt_diag.cuh    pure-store bandwidth probes (measurement only)
//   vmt_posmma.cuh  tcgen05 positioning GEMM, co-resident with the generation kernel
#pragma once

#include "vmt_common.cuh"
#include "vmt_gen.cuh"
#include "vmt_jump.cuh"
#include "vmt_matrix.cuh"
#include "vmt_diag.cuh"
#include "vmt_posmma.cuh"
