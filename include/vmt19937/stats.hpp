// vmt19937/stats.hpp -- statistical smoke tests, source-compatible with the
// reference's proj/include/vmt19937/stats.hpp:13-50.
//
// These overloads take caller callbacks (WordSource), so the words arrive one
// at a time on the host: the header counts them there and the library
// evaluates the statistic with the reference's formulas
// (vmt_monobit_from_counts, vmt_chi2_bytes_from_counts,
// vmt_lane_cross_correlation_from_words). For a generator's own stream use
// the fused GPU consumers instead (vmt_monobit / vmt_chi2_bytes on a handle,
// VmtGenerator::monobit / chi2_bytes), which count inside the generation
// kernel and never store the words.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "vmt19937/detail/abi.hpp"

namespace vmt19937 {

struct StatReport {
    std::string name;
    std::uint64_t samples = 0;
    double statistic = 0.0;
    double p_value = 0.0;
    bool pass = false;
};

inline constexpr double kSignificance = 0.001;

using WordSource = std::function<std::uint32_t()>;

namespace detail {
inline StatReport to_report(const vmt_stat_report& r) {
    StatReport s;
    s.name = r.name ? r.name : "";
    s.samples = r.samples;
    s.statistic = r.statistic;
    s.p_value = r.p_value;
    s.pass = r.pass != 0;
    return s;
}

inline double regularized_gamma_q(double a, double x) {
    double q = 0.0;
    check(vmt_regularized_gamma_q(a, x, &q));
    return q;
}
} // namespace detail

// stats.cpp:65-81
inline StatReport monobit(const WordSource& source, std::uint64_t count) {
    if (count < 1000000)
        throw std::invalid_argument("monobit needs at least 10^6 words");
    std::uint64_t ones = 0;
    for (std::uint64_t i = 0; i < count; ++i)
        ones += std::uint64_t(__builtin_popcount(source()));
    vmt_stat_report r{};
    detail::check(vmt_monobit_from_counts(count, ones, &r));
    return detail::to_report(r);
}

// stats.cpp:83-107
inline StatReport chi2_bytes(const WordSource& source, std::uint64_t count) {
    if (count * 4 < 256 * 50)
        throw std::invalid_argument("chi2_bytes needs at least 50 expected bytes per bin");
    std::vector<std::uint64_t> bins(256, 0);
    for (std::uint64_t i = 0; i < count; ++i) {
        const std::uint32_t w = source();
        for (int b = 0; b < 4; ++b)
            ++bins[(w >> (8 * b)) & 0xFFu];
    }
    vmt_stat_report r{};
    detail::check(vmt_chi2_bytes_from_counts(count, bins.data(), &r));
    return detail::to_report(r);
}

// stats.cpp:109-150 (sources drained lane by lane, like the reference)
inline StatReport lane_cross_correlation(const std::vector<WordSource>& lanes, std::uint64_t count) {
    const std::size_t m = lanes.size();
    if (m < 2)
        throw std::invalid_argument("lane_cross_correlation needs at least 2 lanes");
    std::vector<std::uint32_t> words(m * count);
    for (std::size_t t = 0; t < m; ++t)
        for (std::uint64_t i = 0; i < count; ++i)
            words[i * m + t] = lanes[t]();
    vmt_stat_report r{};
    detail::check(vmt_lane_cross_correlation_from_words(words.data(), unsigned(m), count, &r));
    return detail::to_report(r);
}

} // namespace vmt19937
