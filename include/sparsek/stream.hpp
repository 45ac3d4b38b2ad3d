// sparsek/stream.hpp — drop-in for proj/include/sparsek/stream.hpp:12-83.
// StreamState is device-resident (skb_stream_*): the survivors and saturated
// entries live as two device arrays sorted by (value desc, index asc); push
// runs the reference's push/scan arithmetic in one warp (tau bit-identical,
// proj/src/stream.cpp:72-152) and returns the step result in one round trip.
// Capacity grows transparently (the state is moved through the reference's
// own wire format).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "sparsek/detail/device.hpp"
#include "sparsek/selection.hpp"
#include "sparsek/sparsek_op.hpp"

namespace sparsek {

struct StreamStepResult {
    double tau = kNegInf;
    std::size_t t = 0;
    bool inserted = false;
    std::vector<std::size_t> evicted;
    bool cap_forced = false;
};

class StreamState {
  public:
    explicit StreamState(KBudget k, std::size_t heap_cap = 0) : k_(k.k) {
        skb_stream* s = nullptr;
        detail::check(skb_stream_create(k.k, (int64_t)heap_cap, kInitialCapacity, &s));
        h_.reset(s, skb_stream_destroy);
        cap_ = kInitialCapacity;
    }
    StreamState(const StreamState& o) : k_(o.k_) { adopt_blob(o.blob(), std::max<int64_t>(o.cap_, 1)); }
    StreamState& operator=(const StreamState& o) {
        if (this != &o) {
            k_ = o.k_;
            adopt_blob(o.blob(), std::max<int64_t>(o.cap_, 1));
        }
        return *this;
    }
    StreamState(StreamState&&) noexcept = default;
    StreamState& operator=(StreamState&&) noexcept = default;

    StreamStepResult push(double z_t) {
        if (!std::isfinite(z_t)) throw NumericError("stream_push: non-finite value");
        if ((int64_t)t_ >= cap_) grow();
        skb_stream_step st{};
        ev_.resize((size_t)cap_);
        detail::check(skb_stream_push_step(h_.get(), z_t, &st, ev_.data(), (int64_t)ev_.size(), nullptr));
        StreamStepResult r;
        r.tau = st.tau;
        r.t = (std::size_t)st.t;
        r.inserted = st.inserted != 0;
        r.cap_forced = st.cap_forced != 0;
        r.evicted.assign(ev_.begin(), ev_.begin() + st.n_evicted);
        t_ = r.t;
        return r;
    }

    SparseKSolution solution() const {
        const skb_stream_info in = info();
        const size_t n = (size_t)std::max<int64_t>(in.survivors, 1);
        detail::Buf dp(n * 8), di(n * 8);
        skb_stream_solution_info si{};
        detail::check(skb_stream_solution(h_.get(), dp.as<double>(), di.as<int64_t>(), nullptr, &si, nullptr));
        SparseKSolution sol;
        sol.p = dp.to_host<double>((size_t)si.n);
        const std::vector<int64_t> idx = di.to_host<int64_t>((size_t)si.n);
        sol.indices.assign(idx.begin(), idx.end());
        sol.tau = si.infeasible ? kNegInf : si.tau;
        sol.infeasible = si.infeasible != 0;
        sol.degenerate = si.degenerate != 0;
        sol.u_count = (std::size_t)si.u_count;
        sol.w_count = (std::size_t)si.w_count;
        detail::classify(sol);
        return sol;
    }

    double tau() const { return info().tau; }
    std::size_t t() const { return (std::size_t)info().t; }
    double k() const { return k_; }
    std::size_t survivor_count() const { return (std::size_t)info().survivors; }
    std::size_t saturated_count() const { return (std::size_t)info().saturated; }
    bool is_evicted(std::size_t index) const {
        const skb_stream_info in = info();
        std::vector<uint8_t> ev((size_t)std::max<int64_t>(in.t, 1));
        detail::check(skb_stream_survivors(h_.get(), nullptr, nullptr, ev.data(), nullptr));
        return ev.at(index) != 0;
    }
    std::uint64_t cap_drops() const { return info().cap_drops; }
    std::uint64_t total_heap_ops() const { return info().heap_ops; }
    double sum_drift() const { return 0.0; }  // sums are re-derived on the device

    struct Entry {
        double value;
        std::size_t index;
    };
    std::vector<Entry> survivors_raw() const {
        const skb_stream_info in = info();
        std::vector<double> v((size_t)std::max<int64_t>(in.survivors, 1));
        std::vector<int64_t> ix(v.size());
        detail::check(skb_stream_survivors(h_.get(), v.data(), ix.data(), nullptr, nullptr));
        std::vector<Entry> out((size_t)in.survivors);
        for (size_t i = 0; i < out.size(); ++i) out[i] = {v[i], (std::size_t)ix[i]};
        return out;
    }

    void serialize(std::vector<std::uint8_t>& out) const {
        const std::vector<std::uint8_t> b = blob();
        out.insert(out.end(), b.begin(), b.end());
    }
    static StreamState deserialize(const std::uint8_t* data, std::size_t len, std::size_t* used) {
        StreamState s;
        s.adopt_blob(std::vector<std::uint8_t>(data, data + len), 0);
        if (used) *used = s.blob().size();
        return s;
    }

    skb_stream* handle() const { return h_.get(); }

  private:
    static constexpr int64_t kInitialCapacity = 1 << 14;
    StreamState() = default;
    skb_stream_info info() const {
        skb_stream_info in{};
        detail::check(skb_stream_query(h_.get(), &in, nullptr));
        return in;
    }
    std::vector<std::uint8_t> blob() const {
        size_t n = 0;
        detail::check(skb_stream_serialize(h_.get(), nullptr, &n, nullptr));
        std::vector<std::uint8_t> b(n);
        detail::check(skb_stream_serialize(h_.get(), b.data(), &n, nullptr));
        b.resize(n);
        return b;
    }
    void adopt_blob(const std::vector<std::uint8_t>& b, int64_t cap) {
        // the blob's push count sets the minimum capacity (u64 at byte 24)
        uint64_t t = 0;
        if (b.size() >= 32)
            for (int i = 0; i < 8; ++i) t |= (uint64_t)b[24 + i] << (8 * i);
        cap = std::max<int64_t>({cap, (int64_t)t * 2, kInitialCapacity});
        skb_stream* s = nullptr;
        detail::check(skb_stream_deserialize(b.data(), b.size(), cap, &s));
        h_.reset(s, skb_stream_destroy);
        cap_ = cap;
        t_ = (std::size_t)t;
        skb_stream_info in{};
        detail::check(skb_stream_query(s, &in, nullptr));
        k_ = in.k;
    }
    void grow() { adopt_blob(blob(), cap_ * 4); }

    double k_ = 0.0;
    std::shared_ptr<skb_stream> h_;
    int64_t cap_ = 0;
    std::size_t t_ = 0;
    std::vector<int64_t> ev_;
};

inline StreamState stream_init(KBudget k) { return StreamState(k); }

inline SparseKSolution stream_push(StreamState& state, double z_t) {
    state.push(z_t);
    return state.solution();
}

// stream.cpp:199-222, computed on the device (skb_stream_solution's hard flag).
inline SelectionMask stream_mask(const StreamState& state) {
    if (state.t() == 0) throw ArgumentError("stream_mask: empty state");
    const std::size_t n = std::max<std::size_t>(state.survivor_count(), 1);
    detail::Buf dp(n * 8), di(n * 8), dh(n);
    skb_stream_solution_info si{};
    detail::check(skb_stream_solution(state.handle(), dp.as<double>(), di.as<int64_t>(), dh.as<uint8_t>(), &si, nullptr));
    SelectionMask m;
    m.mode = SelectionMask::Mode::soft;
    m.soft = dp.to_host<double>((size_t)si.n);
    const std::vector<int64_t> idx = di.to_host<int64_t>((size_t)si.n);
    const std::vector<uint8_t> hard = dh.to_host<uint8_t>((size_t)si.n);
    m.hard.assign((size_t)si.n, 0.0);
    for (size_t i = 0; i < (size_t)si.n; ++i)
        if (hard[i]) {
            m.hard[i] = 1.0;
            m.indices.push_back((std::size_t)idx[i]);
        }
    return m;
}

}  // namespace sparsek
