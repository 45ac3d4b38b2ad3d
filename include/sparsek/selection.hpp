// sparsek/selection.hpp — drop-in for proj/include/sparsek/selection.hpp:13-107.
// score_tokens runs K1 on the GPU (skb_score_continue: float64 dot products and
// the reference's sequential Welford arithmetic, bit-identical u).
#pragma once

#include <cmath>
#include <cstddef>
#include <vector>

#include "sparsek/common.hpp"
#include "sparsek/numerics.hpp"
#include "sparsek/sparsek_op.hpp"

namespace sparsek {

enum class NormMode { none, timestep_norm };
enum class SlopeOrder { slope_then_norm, norm_then_slope };

struct ScoringParams {
    std::vector<double> w_score;
    double slope_eps = 0.01;
    bool slope_enabled = true;
    NormMode norm_mode = NormMode::timestep_norm;
    SlopeOrder slope_order = SlopeOrder::norm_then_slope;

    void validate() const {
        if (!(slope_eps > 0.0)) throw ArgumentError("ScoringParams: slope_eps must be positive");
        for (double v : w_score)
            if (!std::isfinite(v)) throw NumericError("ScoringParams: non-finite w_score");
    }
};

struct TimestepNormState {
    std::size_t count = 0;
    double mean = 0.0;
    double m2 = 0.0;
    double eps = 1e-5;

    double push(double r) {  // selection.cpp:13-20 (the state object's own update)
        if (!std::isfinite(r)) throw NumericError("timestep_norm: non-finite input");
        ++count;
        const double delta = r - mean;
        mean += delta / static_cast<double>(count);
        m2 += delta * (r - mean);
        return (r - mean) / std::sqrt(variance() + eps);
    }
    double variance() const { return count ? m2 / static_cast<double>(count) : 0.0; }
};

struct SelectionMask {
    enum class Mode { hard, soft, straight_through };
    std::vector<double> hard;
    std::vector<double> soft;
    std::vector<std::size_t> indices;
    Mode mode = Mode::hard;
};

namespace detail {
inline skb_scoring to_c(const ScoringParams& p) {
    skb_scoring s{};
    s.norm_mode = p.norm_mode == NormMode::timestep_norm ? 1 : 0;
    s.slope_order = p.slope_order == SlopeOrder::norm_then_slope ? 1 : 0;
    s.slope_enabled = p.slope_enabled ? 1 : 0;
    s.chunk_len = 0;
    s.slope_eps = p.slope_eps;
    return s;
}
}  // namespace detail

// Scores of the rows of x continuing `norm` (selection.cpp:22-31). The device
// continues the position count from the norm state, so under timestep_norm
// base_pos must equal norm.count (how the reference's engine always calls it).
inline std::vector<double> score_tokens(const Tensor2& x, const ScoringParams& params, TimestepNormState& norm,
                                        std::size_t base_pos = 0) {
    params.validate();
    if (x.cols != params.w_score.size()) throw ShapeError("score_tokens: x.cols != w_score length");
    if (params.norm_mode == NormMode::timestep_norm && base_pos != norm.count)
        throw ArgumentError("score_tokens: base_pos must equal the norm state's count (device continuation)");
    if (x.rows == 0) return {};
    const skb_scoring sc = detail::to_c(params);
    std::vector<double> st = {params.norm_mode == NormMode::timestep_norm ? (double)norm.count : (double)base_pos,
                              norm.mean, norm.m2};
    detail::Buf dx(x.data), dw(params.w_score), ds(st), draw(x.rows * 8), du(x.rows * 8);
    detail::check(skb_score_continue(1, (int64_t)x.rows, (int64_t)x.cols, SKB_F64, dx.get(), dw.as<double>(), &sc,
                                     ds.as<double>(), draw.as<double>(), du.as<double>(), nullptr));
    if (params.norm_mode == NormMode::timestep_norm) {
        const std::vector<double> s2 = ds.to_host<double>(3);
        norm.count = (std::size_t)s2[0];
        norm.mean = s2[1];
        norm.m2 = s2[2];
    }
    return du.to_host<double>(x.rows);
}

}  // namespace sparsek
