// C ABI of the fused statistics consumer (included by vmt_capi.cu): the
// reference's monobit and chi2_bytes smoke tests (stats.cpp:65-107) over a
// generator's stream, with the counts taken by the generation kernel in
// MODE_STATS (nothing is stored) and the statistics evaluated on the host by
// the reference's formulas, operation for operation.
#include <cmath>

namespace {

constexpr double kSignificance = 0.001; // stats.hpp:24

// Regularized upper incomplete gamma Q(a, x) (stats.cpp:13-60): lower-tail
// series below a+1, modified-Lentz continued fraction above. The reference's
// canonical build (-O3 -march=native, CMakeLists.txt:14-21) contracts
// a*b+c into fused multiply-adds; std::fma reproduces those roundings.
// Returns Q = 1 - P directly: the reference inlines the series into its
// caller and contracts 1 - sum*e into one fused negative multiply-add.
double gamma_q_series(double a, double x) {
    double term = 1.0 / a;
    double sum = term;
    for (int n = 1; n < 10000; ++n) {
        term *= x / (a + n);
        sum += term;
        if (std::abs(term) < std::abs(sum) * 1e-17)
            break;
    }
    return std::fma(-sum, std::exp(std::fma(a, std::log(x), -x) - std::lgamma(a)), 1.0);
}

double gamma_q_cf(double a, double x) {
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 10000; ++i) {
        const double an = -double(i) * (double(i) - a);
        b += 2.0;
        d = std::fma(an, d, b);
        if (std::abs(d) < tiny)
            d = tiny;
        c = b + an / c;
        if (std::abs(c) < tiny)
            c = tiny;
        d = 1.0 / d;
        const double delta = d * c;
        h *= delta;
        if (std::abs(delta - 1.0) < 1e-17)
            break;
    }
    return h * std::exp(std::fma(a, std::log(x), -x) - std::lgamma(a));
}

double regularized_gamma_q(double a, double x) {
    if (a <= 0.0 || x < 0.0)
        throw std::invalid_argument("regularized_gamma_q domain");
    if (x == 0.0)
        return 1.0;
    if (x < a + 1.0)
        return gamma_q_series(a, x);
    return gamma_q_cf(a, x);
}

void count_word(std::uint32_t w, std::uint64_t* c) {
    c[0] += (std::uint64_t)__builtin_popcount(w);
    c[1 + (w & 0xFFu)] += 1;
    c[1 + ((w >> 8) & 0xFFu)] += 1;
    c[1 + ((w >> 16) & 0xFFu)] += 1;
    c[1 + (w >> 24)] += 1;
}

// Consumes the next n words of h like a fill: c[0] = one bits, c[1+b] =
// occurrences of byte value b (4 bytes per word).
void stat_counts(vmt_generator* h, std::uint64_t n, std::uint64_t* c, cudaStream_t st) {
    std::fill(c, c + kStatWords, 0ull);
    if (h->pos < h->gpos) { // words already staged for single / block16 queries
        const std::uint64_t take = std::min<std::uint64_t>(n, h->gpos - h->pos);
        for (std::uint64_t i = 0; i < take; ++i)
            count_word(h->hstage[h->pos - h->hstage_start + i], c);
        h->pos += take;
        n -= take;
    }
    if (n) {
        h->stat_out.reserve(kStatWords);
        gpu_generate(h, MODE_STATS, nullptr, n, st, h->stat_out.p);
        std::vector<unsigned long long> g(kStatWords);
        VMT_CUDA(cudaMemcpyAsync(g.data(), h->stat_out.p, kStatWords * 8, cudaMemcpyDeviceToHost, st));
        VMT_CUDA(cudaStreamSynchronize(st));
        for (int j = 0; j < kStatWords; ++j)
            c[j] += g[j];
        h->pos = h->gpos;
    }
    h->mark(st);
}

// lane_cross_correlation's arithmetic (stats.cpp:109-150) over count*m words
// in combined-stream order (lane t's i-th word at words[i*m + t]).
void lane_corr(const std::uint32_t* words, unsigned m, std::uint64_t count, vmt_stat_report* out) {
    std::vector<double> u((std::size_t)(count * m)); // [t][i]
    for (std::uint64_t i = 0; i < count; ++i)
        for (unsigned t = 0; t < m; ++t)
            u[t * count + i] = (double(words[i * m + t]) + 0.5) / 4294967296.0;
    std::vector<double> mean(m, 0.0), var(m, 0.0);
    for (unsigned t = 0; t < m; ++t) {
        const double* x = u.data() + t * count;
        for (std::uint64_t i = 0; i < count; ++i)
            mean[t] += x[i];
        mean[t] /= double(count);
        for (std::uint64_t i = 0; i < count; ++i)
            var[t] += (x[i] - mean[t]) * (x[i] - mean[t]);
    }
    double max_rho = 0.0;
    for (unsigned s = 0; s < m; ++s)
        for (unsigned t = s + 1; t < m; ++t) {
            const double* a = u.data() + s * count;
            const double* b = u.data() + t * count;
            double cov = 0.0;
            for (std::uint64_t i = 0; i < count; ++i)
                cov += (a[i] - mean[s]) * (b[i] - mean[t]);
            const double denom = std::sqrt(var[s] * var[t]);
            const double rho = denom > 0.0 ? cov / denom : 1.0;
            max_rho = std::max(max_rho, std::abs(rho));
        }
    out->name = "lane_cross_correlation";
    out->samples = count;
    out->statistic = max_rho;
    out->p_value = std::erfc(max_rho * std::sqrt(double(count)) / std::sqrt(2.0));
    out->pass = max_rho < 4.0 / std::sqrt(double(count));
}

} // namespace

extern "C" {

int vmt_stat_counts(vmt_handle h, uint64_t n, uint64_t* out257, void* stream) {
    return guarded([&] {
        require(h && out257, VMT_EINVAL, "null argument");
        DeviceGuard g(h->device);
        stat_counts(h, n, out257, h->pick(stream));
    });
}

int vmt_regularized_gamma_q(double a, double x, double* out) {
    return guarded([&] {
        require(out != nullptr, VMT_EINVAL, "null argument");
        *out = regularized_gamma_q(a, x);
    });
}

int vmt_monobit_from_counts(uint64_t count, uint64_t ones, vmt_stat_report* out) {
    return guarded([&] {
        require(out != nullptr, VMT_EINVAL, "null argument");
        if (count < 1000000)
            throw std::invalid_argument("monobit needs at least 10^6 words");
        const double nbits = double(count) * 32.0;
        const double excess = 2.0 * double((std::int64_t)ones) - nbits; // ones - zeros
        const double z = excess / std::sqrt(nbits);
        out->name = "monobit";
        out->samples = count;
        out->statistic = z;
        out->p_value = std::erfc(std::abs(z) / std::sqrt(2.0));
        out->pass = out->p_value >= kSignificance;
    });
}

int vmt_chi2_bytes_from_counts(uint64_t count, const uint64_t* bins256, vmt_stat_report* out) {
    return guarded([&] {
        require(out != nullptr && bins256 != nullptr, VMT_EINVAL, "null argument");
        if (count * 4 < 256 * 50)
            throw std::invalid_argument("chi2_bytes needs at least 50 expected bytes per bin");
        const double expected = double(count) * 4.0 / 256.0;
        double stat = 0.0;
        for (int b = 0; b < 256; ++b) {
            const double d = double(bins256[b]) - expected;
            stat += d * d / expected;
        }
        out->name = "chi2_bytes";
        out->samples = count;
        out->statistic = stat;
        out->p_value = regularized_gamma_q(255.0 / 2.0, stat / 2.0);
        out->pass = out->p_value >= kSignificance / 2.0 && out->p_value <= 1.0 - kSignificance / 2.0;
    });
}

int vmt_monobit(vmt_handle h, uint64_t count, vmt_stat_report* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        if (count < 1000000)
            throw std::invalid_argument("monobit needs at least 10^6 words");
        DeviceGuard g(h->device);
        std::uint64_t c[kStatWords];
        stat_counts(h, count, c, h->pick(nullptr));
        const int rc = vmt_monobit_from_counts(count, c[0], out);
        if (rc != VMT_OK)
            throw VmtError(rc, g_last_error);
    });
}

int vmt_chi2_bytes(vmt_handle h, uint64_t count, vmt_stat_report* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        if (count * 4 < 256 * 50)
            throw std::invalid_argument("chi2_bytes needs at least 50 expected bytes per bin");
        DeviceGuard g(h->device);
        std::uint64_t c[kStatWords];
        stat_counts(h, count, c, h->pick(nullptr));
        const int rc = vmt_chi2_bytes_from_counts(count, c + 1, out);
        if (rc != VMT_OK)
            throw VmtError(rc, g_last_error);
    });
}

// lane_cross_correlation (stats.cpp:109-150) over the next count*L words of h:
// column t of the combined stream is lane t's own output sequence (SURVEY.md
// A13), which is what the CLI feeds it for a fresh generator
// (vmt19937_main.cpp:216-229). Host arithmetic in the reference's order; the
// reference build's partly vectorised, partly fused sums differ from it in
// the last bits (floating point: parity within 1e-12 relative).
int vmt_lane_cross_correlation(vmt_handle h, uint64_t count, vmt_stat_report* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        const unsigned m = h->L;
        if (m < 2)
            throw std::invalid_argument("lane_cross_correlation needs at least 2 lanes");
        std::vector<std::uint32_t> words((std::size_t)(count * m));
        if (count) {
            const int rc = vmt_fill_u32(h, words.data(), count * m, nullptr);
            if (rc != VMT_OK)
                throw VmtError(rc, g_last_error);
        }
        lane_corr(words.data(), m, count, out);
    });
}

int vmt_lane_cross_correlation_from_words(const uint32_t* words, unsigned lanes, uint64_t count,
                                          vmt_stat_report* out) {
    return guarded([&] {
        require(out != nullptr && (words != nullptr || count == 0), VMT_EINVAL, "null argument");
        if (lanes < 2)
            throw std::invalid_argument("lane_cross_correlation needs at least 2 lanes");
        lane_corr(words, lanes, count, out);
    });
}

} // extern "C"
