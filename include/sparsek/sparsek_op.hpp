// sparsek/sparsek_op.hpp — drop-in for proj/include/sparsek/sparsek_op.hpp:13-66.
// The projection is solved on the GPU (skb_sparsek: sort-free 32-ary
// breakpoint search per row); the index sets are read back with p.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <vector>

#include "sparsek/detail/device.hpp"
#include "sparsek/numerics.hpp"

namespace sparsek {

struct KBudget {
    double k;
    explicit KBudget(double kk) : k(kk) {
        if (!(kk > 0.0) || !std::isfinite(kk)) throw ArgumentError("KBudget: k must be positive and finite");
    }
};

struct SparseKSolution {
    std::vector<double> p;
    double tau = kNegInf;
    std::size_t u_count = 0;
    std::size_t w_count = 0;
    std::vector<std::size_t> support;   // 0 < p < 1, ascending
    std::vector<std::size_t> full_set;  // p == 1, ascending
    bool degenerate = false;
    bool infeasible = false;
    std::vector<std::size_t> indices;   // stream results: slot -> original position
};

namespace detail {
inline void check_finite(const std::vector<double>& z, const char* who) {
    for (double v : z)
        if (!std::isfinite(v)) throw NumericError(std::string(who) + ": non-finite input");
}
// p (on the host) -> support / full_set, as finish() classifies (sparsek_op.cpp:36-57)
inline void classify(SparseKSolution& s) {
    s.support.clear();
    s.full_set.clear();
    for (std::size_t j = 0; j < s.p.size(); ++j) {
        if (s.p[j] == 1.0) s.full_set.push_back(j);
        else if (s.p[j] > 0.0) s.support.push_back(j);
    }
}
inline SparseKSolution solve_device(const std::vector<double>& z, double k) {
    const std::size_t m = z.size();
    Buf dz(z), dp(m * 8), dt(8), du(8), dw(8), df(4);
    check(skb_sparsek(1, (int64_t)m, dz.as<double>(), k, dp.as<double>(), dt.as<double>(), du.as<int64_t>(),
                      dw.as<int64_t>(), df.as<int32_t>(), nullptr));
    SparseKSolution s;
    s.p = dp.to_host<double>(m);
    s.tau = dt.to_host<double>(1)[0];
    s.u_count = (std::size_t)du.to_host<int64_t>(1)[0];
    s.w_count = (std::size_t)dw.to_host<int64_t>(1)[0];
    const int32_t fl = df.to_host<int32_t>(1)[0];
    s.degenerate = (fl & 1) != 0;
    s.infeasible = (fl & 2) != 0;
    classify(s);
    return s;
}
}  // namespace detail

inline SparseKSolution sparsek(const std::vector<double>& z, KBudget k) {
    if (z.empty()) throw ArgumentError("sparsek: empty input");
    detail::check_finite(z, "sparsek");
    return detail::solve_device(z, k.k);
}

struct PartialSortStats {
    std::uint64_t calls = 0;
    std::uint64_t fallbacks = 0;
};

// The device always evaluates the exact projection — what both branches of
// the reference return. `stats` counts the calls and the reference's
// fallbacks: its truncated scan cannot certify exactly when the accepted
// support reaches the cap (w_count >= sort_cap).
inline SparseKSolution sparsek_partial(const std::vector<double>& z, KBudget k, std::size_t sort_cap,
                                       PartialSortStats* stats = nullptr) {
    if (z.empty()) throw ArgumentError("sparsek_partial: empty input");
    if (static_cast<double>(sort_cap) < std::ceil(k.k)) throw ArgumentError("sparsek_partial: sort_cap below ceil(k)");
    if (stats) ++stats->calls;
    detail::check_finite(z, "sparsek_partial");
    SparseKSolution s = detail::solve_device(z, k.k);
    if (stats && !s.infeasible && sort_cap < z.size() && s.w_count >= sort_cap) ++stats->fallbacks;
    return s;
}

inline std::vector<double> sparsek_jvp(const SparseKSolution& sol, const std::vector<double>& v) {
    if (v.size() != sol.p.size()) throw ShapeError("sparsek_jvp: v length mismatch");
    std::vector<double> out(v.size(), 0.0);
    if (v.empty()) return out;
    detail::Buf dp(sol.p), dv(v), dout(v.size() * 8);
    detail::check(skb_support_jvp((int64_t)v.size(), dp.as<double>(), dv.as<double>(), dout.as<double>(), nullptr));
    return dout.to_host<double>(v.size());
}

inline std::vector<double> topk_hard(const std::vector<double>& z, std::size_t k) {
    const std::size_t m = z.size();
    if (k >= m) return std::vector<double>(m, 1.0);
    if (k == 0) return std::vector<double>(m, 0.0);
    detail::Buf dz(z), dout(m * 8);
    detail::check(skb_topk_hard(1, (int64_t)m, dz.as<double>(), (int64_t)k, dout.as<double>(), nullptr));
    return dout.to_host<double>(m);
}

struct StResult {
    std::vector<double> forward;
    SparseKSolution backward_carrier;
};

inline StResult sparsek_st(const std::vector<double>& z, KBudget k) {
    StResult r;
    r.backward_carrier = sparsek(z, k);
    r.forward = topk_hard(z, static_cast<std::size_t>(std::floor(k.k)));
    return r;
}

}  // namespace sparsek
