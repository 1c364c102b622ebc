// C ABI of the generator batch (config 3) and the single-process multi-GPU
// fill (config 4) -- SURVEY.md 8b `vmt_batch_create / vmt_batch_fill_u32` and
// `vmt_multi_gpu_fill`. Included by vmt_capi.cu (same translation unit).

struct vmt_batch {
    int device = 0;
    unsigned L = 1, ngen = 0, q = 0;
    std::uint64_t bw = 624;
    std::uint64_t pos = 0;       // words consumed per generator (all in lockstep)
    std::uint64_t cur_block = 0; // block the states in `cur` are at
    cudaStream_t own = nullptr;
    DevBuf<std::uint32_t> cur, next, scratch; // [ngen][624][L]
    DevBuf<std::uint64_t> polys;
    Counters cnt;
};

namespace {

// n words of every generator from position h->pos into out (device),
// generator-major with stride n.
void batch_generate(vmt_batch* h, std::uint32_t* out, std::uint64_t n, cudaStream_t st) {
    const std::uint64_t P0 = h->pos, P1 = h->pos + n;
    const std::uint64_t b0 = P0 / h->bw, b1 = (P1 + h->bw - 1) / h->bw;
    if (h->cur_block != b0) { // a skip moved the position: jump every lane state
        Gf2Field& F = Gf2Field::instance();
        const std::uint64_t delta = b0 - h->cur_block;
        const unsigned __int128 d = (unsigned __int128)delta * kN;
        const Poly p = F.x_pow128((std::uint64_t)d, (std::uint64_t)(d >> 64));
        h->polys.reserve(kPolyWords);
        VMT_CUDA(cudaMemcpyAsync(h->polys.p, p.data(), kPolyWords * 8, cudaMemcpyHostToDevice, st));
        AffineJobs a;
        a.n = (int)(h->ngen * h->L);
        a.div = (int)h->L;
        a.s_a = (long long)kN * h->L;
        a.s_b = 1;
        a.d_a = (long long)kN * h->L;
        a.d_b = 1;
        launch_jumps_affine(st, h->cur.p, (int)h->L, h->next.p, (int)h->L, h->polys.p, a, h->cnt);
        h->cur.swap(h->next);
        h->cur_block = b0;
    }
    const Variant& v = pick_variant(h->L, 0);
    const int V = v.G >= v.VW ? v.VW : v.G;
    const std::uintptr_t addr = reinterpret_cast<std::uintptr_t>(out);
    const bool vec = addr % 4 == 0 && ((addr / 4 - P0) % V == 0) && (P0 % V == 0) && (n % V == 0);
    GenFn fn = v.fn[MODE_U32][vec ? 1 : 0];
    prepare_gen(h->device, fn, v.NT, v.smem[MODE_U32]);
    GenParams p{};
    p.chunk_states = h->cur.p;
    p.out = out;
    p.save_state = h->next.p;
    p.first_block = b0;
    p.end_block = b1;
    p.pos_begin = P0;
    p.pos_end = P1;
    p.save_block = P1 / h->bw;
    p.out_chunk_stride = n;
    p.blocks_per_chunk = (unsigned)(b1 - b0);
    p.lanes = h->L;
    fn<<<h->ngen * (unsigned)(v.L / v.G), v.NT, v.smem[MODE_U32], st>>>(p);
    VMT_CUDA(cudaGetLastError());
    h->cnt.gen += 1;
    h->cur.swap(h->next);
    h->cur_block = P1 / h->bw;
    h->pos = P1;
}

} // namespace

extern "C" {

int vmt_batch_create(uint32_t seed0, unsigned ngen, unsigned lanes, unsigned jump_exponent, int device,
                     vmt_batch_handle* out) {
    return guarded([&] {
        require(out != nullptr, VMT_EINVAL, "null handle pointer");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        require(ngen > 0 && ngen <= (1u << 20), VMT_EINVAL, "ngen must be in 1..2^20");
        check_device(device);
        std::unique_ptr<vmt_batch> h(new vmt_batch());
        h->device = device;
        h->L = lanes;
        h->ngen = ngen;
        h->bw = 624ull * lanes;
        h->q = jump_exponent == VMT_FULL_PERIOD ? vmt_full_period_exponent(lanes) : jump_exponent;
        DeviceGuard g(device);
        VMT_CUDA(cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking));
        h->cur.reserve((std::size_t)ngen * kN * lanes);
        h->next.reserve((std::size_t)ngen * kN * lanes);
        build_dephased(device, h->own, seed0, ngen, lanes, h->q, h->cur.p, h->polys, h->cnt);
        *out = h.release();
    });
}

int vmt_batch_destroy(vmt_batch_handle h) {
    return guarded([&] {
        if (!h)
            return;
        {
            DeviceGuard g(h->device);
            cudaStreamSynchronize(h->own);
            cudaStreamDestroy(h->own);
        }
        delete h;
    });
}

uint64_t vmt_batch_position(vmt_batch_handle h) { return h ? h->pos : 0; }

int vmt_batch_fill(vmt_batch_handle h, uint32_t* dst, uint64_t n_per_gen, void* stream) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        require(dst != nullptr || n_per_gen == 0, VMT_EINVAL, "null destination");
        if (n_per_gen == 0)
            return;
        DeviceGuard g(h->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->own;
        if (is_device_ptr(dst)) {
            batch_generate(h, dst, n_per_gen, st);
        } else {
            h->scratch.reserve((std::size_t)h->ngen * n_per_gen);
            batch_generate(h, h->scratch.p, n_per_gen, st);
            VMT_CUDA(cudaMemcpyAsync(dst, h->scratch.p, (std::size_t)h->ngen * n_per_gen * 4, cudaMemcpyDeviceToHost,
                                     st));
        }
        VMT_CUDA(cudaStreamSynchronize(st));
    });
}

int vmt_batch_skip(vmt_batch_handle h, uint64_t d) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        h->pos += d; // the lane states are jumped lazily by the next fill
    });
}

int vmt_batch_export_state(vmt_batch_handle h, uint32_t* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        require(h->pos % h->bw == 0 && h->cur_block == h->pos / h->bw, VMT_ESTATE,
                "batch state export needs a block boundary reached by a fill");
        DeviceGuard g(h->device);
        VMT_CUDA(cudaMemcpy(out, h->cur.p, (std::size_t)h->ngen * kN * h->L * 4, cudaMemcpyDeviceToHost));
    });
}

int vmt_multi_gpu_fill(uint32_t seed, unsigned lanes, unsigned jump_exponent, uint64_t n, int ngpus,
                       const int* devices, uint32_t* const* dsts, int mode, uint32_t* checksum) {
    return guarded([&] {
        require(ngpus > 0 && devices != nullptr, VMT_EINVAL, "need at least one device");
        require(mode == 0 || mode == 1, VMT_EINVAL, "mode must be 0 (store) or 1 (xor)");
        require(mode == 1 || dsts != nullptr, VMT_EINVAL, "store mode needs one destination per device");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        std::vector<std::uint32_t> parts(ngpus, 0);
        std::vector<int> rcs(ngpus, VMT_OK);
        std::vector<std::string> errs(ngpus);
        std::vector<std::thread> th;
        for (int k = 0; k < ngpus; ++k)
            th.emplace_back([&, k] {
                const std::uint64_t lo = n / ngpus * k + std::min<std::uint64_t>(k, n % ngpus);
                const std::uint64_t cnt = n / ngpus + (std::uint64_t(k) < n % ngpus ? 1 : 0);
                vmt_handle h = nullptr;
                int rc = vmt_create(seed, lanes, jump_exponent, devices[k], &h);
                if (rc == VMT_OK)
                    rc = vmt_seek(h, lo);
                if (rc == VMT_OK && mode == 0 && cnt)
                    rc = vmt_fill_u32(h, dsts[k], cnt, nullptr);
                if (rc == VMT_OK && (mode == 1 || checksum != nullptr)) {
                    if (mode == 0)
                        rc = vmt_seek(h, lo);
                    if (rc == VMT_OK)
                        rc = vmt_checksum_xor(h, cnt, &parts[k], nullptr);
                }
                if (rc == VMT_OK)
                    rc = vmt_synchronize(h);
                if (rc != VMT_OK)
                    errs[k] = g_last_error;
                if (h)
                    vmt_destroy(h);
                rcs[k] = rc;
            });
        for (auto& t : th)
            t.join();
        for (int k = 0; k < ngpus; ++k)
            if (rcs[k] != VMT_OK)
                throw VmtError(rcs[k], "device " + std::to_string(devices[k]) + ": " + errs[k]);
        if (checksum) {
            std::uint32_t x = 0;
            for (auto p : parts)
                x ^= p;
            *checksum = x;
        }
    });
}

} // extern "C"
