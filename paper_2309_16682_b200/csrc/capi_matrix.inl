// C ABI of the GF(2) jump-matrix path (included by vmt_capi.cu, same
// translation unit): jump matrices computed on the GPU, the reference's .vmtj
// file format, vec_mat_mul and matrix-based de-phasing. Kernels in
// vmt_matrix.cuh; reference anchors in include/vmt19937_b200.h.
#include <fstream>

namespace {

constexpr std::size_t kMatBytes = kMatWords * 8;
constexpr std::uint32_t kVmtjVersion = 1;
constexpr std::size_t kVmtjHeader = 20;

void words_to_eff(const std::uint32_t* src, long long state_stride, int word_stride, std::uint32_t* dst, int n,
                  cudaStream_t st) {
    const long long total = (long long)n * kRowHalves;
    vmt_words_to_eff_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(src, state_stride, word_stride, dst, n);
    VMT_CUDA(cudaGetLastError());
}

void eff_to_words(const std::uint32_t* src, std::uint32_t* dst, long long state_stride, int word_stride, int n,
                  cudaStream_t st) {
    const long long total = (long long)n * kN;
    vmt_eff_to_words_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(src, dst, state_stride, word_stride, n);
    VMT_CUDA(cudaGetLastError());
}

void vec_mat(const std::uint64_t* vecs, std::uint64_t n, const std::uint64_t* mat, std::uint64_t* out,
             cudaStream_t st) {
    for (std::uint64_t s0 = 0; s0 < n; s0 += 65535ull * kVmS) {
        const std::uint64_t m = std::min<std::uint64_t>(n - s0, 65535ull * kVmS);
        dim3 grid(kVmGroups, (unsigned)((m + kVmS - 1) / kVmS));
        vmt_vec_mat_kernel<<<grid, kVmThreads, 0, st>>>(vecs + s0 * kRowWords, mat, out + s0 * kRowWords, (int)m);
        VMT_CUDA(cudaGetLastError());
    }
}

// Rows of p(F) (p = x^d mod P, so p(F) = F^d) into rows_dev: row i is the
// effective state of the basis state e_i jumped by d steps (19937 jobs of
// vmt_jump_kernel, in place on the basis states).
void matrix_from_poly(const Poly& p, std::uint64_t* rows_dev, cudaStream_t st, Counters& cnt) {
    int dev = 0;
    VMT_CUDA(cudaGetDevice(&dev));
    DevBuf<std::uint32_t>& states = thread_scratch<std::uint32_t>(dev, 6); // 50 MB, reused
    DevBuf<std::uint64_t>& dp = thread_scratch<std::uint64_t>(dev, 7);
    states.reserve((std::size_t)kDim * kN);
    dp.reserve(kPolyWords);
    VMT_CUDA(cudaMemcpyAsync(dp.p, p.data(), kPolyWords * 8, cudaMemcpyHostToDevice, st));
    VMT_CUDA(cudaMemsetAsync(states.p, 0, (std::size_t)kDim * kN * 4, st));
    vmt_basis_kernel<<<(kDim + 255) / 256, 256, 0, st>>>(states.p, 0, kDim);
    VMT_CUDA(cudaGetLastError());
    AffineJobs a;
    a.n = kDim;
    a.div = 1;
    a.s_a = kN;
    a.d_a = kN;
    launch_jumps_affine(st, states.p, 1, states.p, 1, dp.p, a, cnt);
    words_to_eff(states.p, kN, 1, reinterpret_cast<std::uint32_t*>(rows_dev), kDim, st);
    cnt.other += 2;
    VMT_CUDA(cudaStreamSynchronize(st)); // the scratch is reused by the next call on this thread
}

// rows_out may be host or device memory.
void matrix_to(const Poly& p, std::uint64_t* rows_out, cudaStream_t st) {
    Counters cnt;
    if (is_device_ptr(rows_out)) {
        matrix_from_poly(p, rows_out, st, cnt);
        return;
    }
    DevBuf<std::uint64_t> rows;
    rows.reserve(kMatWords);
    matrix_from_poly(p, rows.p, st, cnt);
    VMT_CUDA(cudaMemcpy(rows_out, rows.p, kMatBytes, cudaMemcpyDeviceToHost));
}

// A device copy of a caller matrix (host or device) -- or the caller's own
// pointer when it already is device memory.
struct DevMatrix {
    DevBuf<std::uint64_t> own;
    const std::uint64_t* p = nullptr;
    DevMatrix(const std::uint64_t* rows, cudaStream_t st) {
        if (is_device_ptr(rows)) {
            p = rows;
            return;
        }
        own.reserve(kMatWords);
        VMT_CUDA(cudaMemcpyAsync(own.p, rows, kMatBytes, cudaMemcpyHostToDevice, st));
        p = own.p;
    }
};

void put_u32(std::ostream& os, std::uint32_t v) {
    const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                                (unsigned char)(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
}

std::uint32_t get_u32(const unsigned char* b) {
    return std::uint32_t(b[0]) | (std::uint32_t(b[1]) << 8) | (std::uint32_t(b[2]) << 16) | (std::uint32_t(b[3]) << 24);
}

// write_jump_matrix_file (jump_file.cpp:117-123): header, payload, through a
// temporary file renamed into place.
void write_vmtj(const std::string& path, const std::uint64_t* rows_host, unsigned exponent) {
    const std::string tmp = path + ".tmp";
    {
        std::ofstream os(tmp, std::ios::binary | std::ios::trunc);
        if (!os)
            throw std::runtime_error("cannot open " + tmp + " for writing");
        os.write("VMTJ", 4);
        put_u32(os, kVmtjVersion);
        put_u32(os, (std::uint32_t)kDim);
        put_u32(os, exponent);
        put_u32(os, 0);
        os.write(reinterpret_cast<const char*>(rows_host), (std::streamsize)kMatBytes); // little-endian host
        os.flush();
        if (!os)
            throw std::runtime_error("write failed: " + tmp);
    }
    if (std::rename(tmp.c_str(), path.c_str()) != 0)
        throw std::runtime_error("cannot rename " + tmp + " to " + path);
}

// read_jump_matrix_file (jump_file.cpp:125-137) with the same checks, in the
// same order; rows_host == nullptr validates the header and size only.
// A well-formed file of another dimension is std::invalid_argument, like
// vec_mat_mul's dimension check (f2_matrix.cpp:120-121).
unsigned read_vmtj(const std::string& path, std::uint64_t* rows_host) {
    std::ifstream is(path, std::ios::binary | std::ios::ate);
    if (!is)
        throw std::runtime_error("cannot open " + path);
    const std::uint64_t size = (std::uint64_t)is.tellg();
    is.seekg(0);
    unsigned char hdr[kVmtjHeader];
    is.read(reinterpret_cast<char*>(hdr), 4);
    if (!is || std::memcmp(hdr, "VMTJ", 4) != 0)
        throw std::runtime_error(path + ": not a jump-matrix file");
    is.read(reinterpret_cast<char*>(hdr + 4), 16);
    if (get_u32(hdr + 4) != kVmtjVersion)
        throw std::runtime_error(path + ": unsupported version");
    const std::uint32_t dim = get_u32(hdr + 8), exponent = get_u32(hdr + 12), reserved = get_u32(hdr + 16);
    if (!is || reserved != 0)
        throw std::runtime_error(path + ": corrupt header");
    if (dim == 0)
        throw std::runtime_error(path + ": zero dimension");
    const std::uint64_t row_words = (dim + 63) / 64;
    if (size != kVmtjHeader + (std::uint64_t)dim * row_words * 8)
        throw std::runtime_error(path + ": payload size mismatch");
    if (dim != (std::uint32_t)kDim)
        throw std::invalid_argument(path + ": matrix dimension " + std::to_string(dim) + ", expected 19937");
    if (rows_host) {
        is.read(reinterpret_cast<char*>(rows_host), (std::streamsize)kMatBytes);
        if (!is)
            throw std::runtime_error("read failed: " + path);
        const std::uint64_t pad = ~0ull << (kDim - 64 * (kRowWords - 1)); // bits 33..63 of the last word
        for (std::size_t r = 0; r < (std::size_t)kDim; ++r)
            if (rows_host[r * kRowWords + kRowWords - 1] & pad)
                throw std::runtime_error(path + ": nonzero padding bits");
    }
    return exponent;
}

// make_dephased_states (jump.cpp:35-53) with a caller matrix B: lane 0 is the
// seeded state, lane t = lane t-1 * B in the effective representation; all
// lanes interleaved into dst [624][L].
void dephase_with_matrix(std::uint32_t seed, unsigned L, const std::uint64_t* mat_dev, std::uint32_t* dst,
                         cudaStream_t st, Counters& cnt) {
    DevBuf<std::uint32_t> dseed;
    dseed.reserve(1);
    VMT_CUDA(cudaMemcpyAsync(dseed.p, &seed, 4, cudaMemcpyHostToDevice, st));
    vmt_seed_kernel<<<1, 32, 0, st>>>(dseed.p, 1, dst, (long long)kN * L, (int)L);
    VMT_CUDA(cudaGetLastError());
    cnt.other += 1;
    if (L > 1) {
        DevBuf<std::uint64_t> v, w;
        v.reserve(kRowWords);
        w.reserve(kRowWords);
        for (unsigned t = 1; t < L; ++t) {
            words_to_eff(dst + (t - 1), 0, (int)L, reinterpret_cast<std::uint32_t*>(v.p), 1, st);
            vec_mat(v.p, 1, mat_dev, w.p, st);
            eff_to_words(reinterpret_cast<const std::uint32_t*>(w.p), dst + t, 0, (int)L, 1, st);
            cnt.other += 3;
        }
        VMT_CUDA(cudaStreamSynchronize(st));
    }
    VMT_CUDA(cudaStreamSynchronize(st));
}

} // namespace

extern "C" {

int vmt_jump_matrix(uint64_t d_lo, uint64_t d_hi, uint64_t* rows, int device, void* stream) {
    return guarded([&] {
        require(rows != nullptr, VMT_EINVAL, "null argument");
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        matrix_to(Gf2Field::instance().x_pow128(d_lo, d_hi), rows, st);
    });
}

int vmt_jump_matrix_pow2(unsigned q, uint64_t* rows, int device, void* stream) {
    return guarded([&] {
        require(rows != nullptr, VMT_EINVAL, "null argument");
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        matrix_to(Gf2Field::instance().x_pow2(q), rows, st);
    });
}

int vmt_write_jump_matrix_file(const char* path, const uint64_t* rows, unsigned exponent) {
    return guarded([&] {
        require(path != nullptr && rows != nullptr, VMT_EINVAL, "null argument");
        if (is_device_ptr(rows)) {
            std::vector<std::uint64_t> host(kMatWords);
            VMT_CUDA(cudaMemcpy(host.data(), rows, kMatBytes, cudaMemcpyDeviceToHost));
            write_vmtj(path, host.data(), exponent);
        } else {
            write_vmtj(path, rows, exponent);
        }
    });
}

int vmt_read_jump_matrix_file(const char* path, uint64_t* rows, unsigned* exponent) {
    return guarded([&] {
        require(path != nullptr, VMT_EINVAL, "null argument");
        const unsigned e = read_vmtj(path, rows);
        if (exponent)
            *exponent = e;
    });
}

int vmt_compute_jump_matrix_file(const char* path, unsigned exponent, int device) {
    return guarded([&] {
        require(path != nullptr, VMT_EINVAL, "null argument");
        check_device(device);
        DeviceGuard g(device);
        std::vector<std::uint64_t> host(kMatWords);
        matrix_to(Gf2Field::instance().x_pow2(exponent), host.data(), cudaStreamPerThread);
        write_vmtj(path, host.data(), exponent);
    });
}

int vmt_vec_mat_mul(const uint64_t* vecs, uint64_t n, const uint64_t* rows, uint64_t* out, int device,
                    void* stream) {
    return guarded([&] {
        require(vecs && rows && out, VMT_EINVAL, "null argument");
        if (n == 0)
            return;
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        DevMatrix m(rows, st);
        DevBuf<std::uint64_t> dv, dout;
        const std::uint64_t* v = vecs;
        if (!is_device_ptr(vecs)) {
            dv.reserve(n * kRowWords);
            VMT_CUDA(cudaMemcpyAsync(dv.p, vecs, n * kRowWords * 8, cudaMemcpyHostToDevice, st));
            v = dv.p;
        }
        const bool out_dev = is_device_ptr(out);
        std::uint64_t* o = out;
        if (!out_dev) {
            dout.reserve(n * kRowWords);
            o = dout.p;
        }
        vec_mat(v, n, m.p, o, st);
        if (!out_dev)
            VMT_CUDA(cudaMemcpyAsync(out, dout.p, n * kRowWords * 8, cudaMemcpyDeviceToHost, st));
        VMT_CUDA(cudaStreamSynchronize(st));
    });
}

int vmt_jump_states_matrix(const uint32_t* src, uint64_t n, const uint64_t* rows, uint32_t* dst, int device,
                           void* stream) {
    return guarded([&] {
        require(src && rows && dst, VMT_EINVAL, "null argument");
        if (n == 0)
            return;
        require(n <= 0x7FFFFFFFull / kN, VMT_EINVAL, "too many states");
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        DevMatrix m(rows, st);
        DevBuf<std::uint32_t> words;
        DevBuf<std::uint64_t> v, w;
        words.reserve(n * kN);
        v.reserve(n * kRowWords);
        w.reserve(n * kRowWords);
        VMT_CUDA(cudaMemcpyAsync(words.p, src, n * kN * 4,
                                 is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        words_to_eff(words.p, kN, 1, reinterpret_cast<std::uint32_t*>(v.p), (int)n, st);
        vec_mat(v.p, n, m.p, w.p, st);
        eff_to_words(reinterpret_cast<const std::uint32_t*>(w.p), words.p, kN, 1, (int)n, st);
        VMT_CUDA(cudaMemcpyAsync(dst, words.p, n * kN * 4,
                                 is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        VMT_CUDA(cudaStreamSynchronize(st));
    });
}

int vmt_create_from_matrix(uint32_t seed, unsigned lanes, const uint64_t* rows, unsigned exponent, int device,
                           vmt_handle* out) {
    return guarded([&] {
        require(out != nullptr, VMT_EINVAL, "null handle pointer");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        require(rows != nullptr || lanes == 1, VMT_EINVAL, "a jump matrix is required for lanes > 1");
        std::unique_ptr<vmt_generator> h(new_handle(lanes, device));
        h->q = exponent;
        DeviceGuard g(device);
        if (lanes == 1) {
            dephase_with_matrix(seed, 1, nullptr, h->base.p, h->own, h->cnt);
        } else {
            DevMatrix m(rows, h->own);
            dephase_with_matrix(seed, lanes, m.p, h->base.p, h->own, h->cnt);
        }
        VMT_CUDA(cudaMemcpyAsync(h->cur.p, h->base.p, (size_t)kN * lanes * 4, cudaMemcpyDeviceToDevice, h->own));
        VMT_CUDA(cudaStreamSynchronize(h->own));
        *out = h.release();
    });
}

int vmt_create_from_file(uint32_t seed, unsigned lanes, const char* path, int device, vmt_handle* out) {
    return guarded([&] {
        require(out != nullptr && path != nullptr, VMT_EINVAL, "null argument");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        std::vector<std::uint64_t> host(kMatWords);
        const unsigned e = read_vmtj(path, host.data());
        const int rc = vmt_create_from_matrix(seed, lanes, host.data(), e, device, out);
        if (rc != VMT_OK)
            throw VmtError(rc, g_last_error);
    });
}

} // extern "C"
