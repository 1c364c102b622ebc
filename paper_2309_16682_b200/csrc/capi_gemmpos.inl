// Steady-state chunk positioning on the tensor cores (included by vmt_capi.cu).
//
// Consecutive fills of the same shape (same chunk count C and blocks per chunk
// B) advance every chunk start by the same block delta D: chunk c of the next
// fill is chunk c of this one jumped by 624*D words -- one and the same GF(2)
// matrix F^(624 D) for all C*L lane states. Instead of C*L polynomial jumps
// (~0.39 us of GPU each), the new states are one integer GEMM
//   new[C*L][19968] = old[C*L][19968] x F^(624 D)[19968][19968]  (mod 2)
// in word-bit coordinates (vmt_matrix.cuh), int8 x int8 -> int32 on the
// tensor cores via cuBLAS (a plain library GEMM), then packed back into
// words. The 400 MB int8 matrix for a delta is built once (19937 basis jumps
// + expansion) when the delta repeats; two deltas are cached (a fill size
// that is not a multiple of the block alternates between two).
#include <cublas_v2.h>

namespace {

constexpr std::uint64_t kGemmMinRows = 2048; // below this the polynomial jumps win
constexpr std::size_t kGemmMatBytes = (std::size_t)kWB * kWB;

struct GemmPos {
    cublasHandle_t blas = nullptr;
    std::map<std::uint64_t, std::unique_ptr<DevBuf<std::int8_t>>> mats; // delta -> F^(624 delta), word-bit
    std::map<std::uint64_t, int> seen;                                   // delta -> transitions observed
    std::list<std::uint64_t> lru;
    DevBuf<std::int8_t> a;
    DevBuf<std::int32_t> prod;
    bool last_valid = false;
    std::uint64_t last_b0 = 0, last_B = 0, last_C = 0;
    ~GemmPos() {
        if (blas)
            cublasDestroy(blas);
    }
};

#define VMT_CUBLAS(x)                                                                                 \
    do {                                                                                              \
        cublasStatus_t s_ = (x);                                                                      \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                              \
            throw VmtError(VMT_ECUDA, std::string(#x) + ": cuBLAS status " + std::to_string((int)s_));  \
    } while (0)

const std::int8_t* gemm_matrix(vmt_generator* h, GemmPos& gp, std::uint64_t delta, cudaStream_t st) {
    auto it = gp.mats.find(delta);
    if (it != gp.mats.end()) {
        gp.lru.remove(delta);
        gp.lru.push_front(delta);
        return it->second->p;
    }
    if (gp.mats.size() >= 2) {
        VMT_CUDA(cudaStreamSynchronize(st));
        gp.mats.erase(gp.lru.back());
        gp.lru.pop_back();
    }
    Gf2Field& F = Gf2Field::instance();
    const unsigned __int128 d = (unsigned __int128)kN * delta;
    DevBuf<std::uint64_t> rows;
    rows.reserve(kMatWords);
    Counters cnt;
    matrix_from_poly(F.x_pow128((std::uint64_t)d, (std::uint64_t)(d >> 64)), rows.p, st, cnt);
    std::unique_ptr<DevBuf<std::int8_t>> m(new DevBuf<std::int8_t>());
    m->reserve(kGemmMatBytes);
    vmt_gemm_matrix_kernel<<<dim3((kWB + 255) / 256, kWB), 256, 0, st>>>(rows.p, m->p);
    VMT_CUDA(cudaGetLastError());
    VMT_CUDA(cudaStreamSynchronize(st)); // rows is released on return
    h->cnt.other += 1;
    const std::int8_t* p = m->p;
    gp.mats[delta] = std::move(m);
    gp.lru.push_front(delta);
    return p;
}

// dst[C][624][L] = src[C][624][L] jumped by 624*delta words, by one GEMM.
void gemm_position(vmt_generator* h, GemmPos& gp, const std::uint32_t* src, std::uint32_t* dst, std::uint64_t rows,
                   std::uint64_t delta, cudaStream_t st) {
    const std::int8_t* mat = gemm_matrix(h, gp, delta, st);
    if (!gp.blas)
        VMT_CUBLAS(cublasCreate(&gp.blas));
    VMT_CUBLAS(cublasSetStream(gp.blas, st));
    gp.a.reserve(rows * kWB);
    gp.prod.reserve(rows * kWB);
    const long long nwords = (long long)rows * kN;
    const unsigned grid = (unsigned)((nwords + 255) / 256);
    vmt_states_to_i8_kernel<<<grid, 256, 0, st>>>(src, (int)h->L, nwords, gp.a.p);
    VMT_CUDA(cudaGetLastError());
    // In cuBLAS's column-major terms: C (m = 19968 output bits, n = rows) =
    // A^T (m x k) * B (k x n) with A = mat stored [out j][in i] (lda = k),
    // B = the state bits stored [row r][in i] (ldb = k), C = prod stored
    // [row r][out j] (ldc = m): prod[r][j] = sum_i bits[r][i] * M[i][j].
    const std::int32_t one = 1, zero = 0;
    VMT_CUBLAS(cublasGemmEx(gp.blas, CUBLAS_OP_T, CUBLAS_OP_N, kWB, (int)rows, kWB, &one, mat, CUDA_R_8I, kWB,
                            gp.a.p, CUDA_R_8I, kWB, &zero, gp.prod.p, CUDA_R_32I, kWB, CUBLAS_COMPUTE_32I,
                            CUBLAS_GEMM_DEFAULT));
    vmt_i32_to_states_kernel<<<grid, 256, 0, st>>>(gp.prod.p, (int)h->L, nwords, dst);
    VMT_CUDA(cudaGetLastError());
    h->cnt.other += 2; // expand + pack (the GEMM itself is cuBLAS's kernel)
    h->cnt.gemm_positionings += 1;
}

} // namespace
