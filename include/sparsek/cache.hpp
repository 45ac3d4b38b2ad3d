// sparsek/cache.hpp — drop-in for proj/include/sparsek/cache.hpp:14-112.
//
// SparseKvCache<T> is the device-resident recurrent state (skb_xcache_*: the
// K5 slot pool of floor(k) + w + 1 rows, the stream as sorted survivor
// arrays, the TimestepNormState). forward_chunk on a fresh cache runs the
// batch kernels over the chunk and keeps only the retained rows; on a
// non-empty cache each row is one generate_step (exit/admit + attention over
// the retained rows) — the reference's row order, so chunked output equals
// unchunked output (proj/tests/test_cache.cpp:34-64). Memory stays bounded by
// floor(k) + w + 1 rows plus O(positions) scores (max_positions, default 2^20).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "sparsek/attention.hpp"
#include "sparsek/detail/device.hpp"
#include "sparsek/stream.hpp"

namespace sparsek {

template <class T>
class SparseKvCache {
  public:
    SparseKvCache(const AttnConfig& cfg, std::size_t d_model, const ScoringParams& scoring,
                  std::size_t max_positions = std::size_t(1) << 20)
        : cfg_(cfg), d_model_(d_model), scoring_(scoring), max_pos_(max_positions) {
        cfg.validate(d_model, scoring);
        skb_x_desc d = detail::x_desc<T>(max_positions, d_model, cfg, scoring);
        if (cfg.linear_mix) d.flags |= SKB_FLAG_LINEAR_MIX;  // the cache carries phi(k) and the prefix state
        skb_xcache* c = nullptr;
        detail::check(skb_xcache_create(&d, &c));
        h_.reset(c, skb_xcache_destroy);
        cap_ = cfg.k > 0.0 ? static_cast<std::size_t>(std::floor(cfg.k)) : 0;
    }

    SparseKvCache(const SparseKvCache&) = delete;  // one owner of the device state
    SparseKvCache& operator=(const SparseKvCache&) = delete;
    SparseKvCache(SparseKvCache&&) noexcept = default;
    SparseKvCache& operator=(SparseKvCache&&) noexcept = default;

    MatT<T> forward_chunk(const MatT<T>& x_chunk, const AttnParams<T>& params, AttnTape<T>* tape = nullptr,
                          const LinearMixParams<T>* lin = nullptr) {
        if (cfg_.linear_mix && !lin) throw ConfigError("forward_chunk: linear mix needs feature parameters");
        if (x_chunk.cols != d_model_) throw ShapeError("forward_chunk: x.cols != d_model");
        detail::check_params(params, d_model_);
        const std::size_t n = x_chunk.rows;
        MatT<T> y(n, d_model_);
        if (n == 0) return y;
        if (tape) {
            // training mode: the tape of a fresh cache's first chunk is
            // sparsek_attention's; later chunks go through chunked_forward
            if (positions_seen() != 0)
                throw ArgumentError("forward_chunk: a tape needs a fresh cache on this backend (use chunked_forward)");
            detail::run_forward(x_chunk, params, scoring_, cfg_, tape, 0, cfg_.linear_mix ? lin : nullptr);
        }
        detail::DeviceParams<T> dp(params, scoring_);
        detail::Buf dx(x_chunk.data), dy(y.data.size() * sizeof(T));
        if (cfg_.linear_mix) {  // Appendix B.1: the mixture readout with the carried prefix state
            detail::Buf df(detail::pack_feat(*lin, cfg_.heads, d_model_ / cfg_.heads));
            detail::check(skb_xcache_forward_chunk_lin(h_.get(), dx.get(), (int64_t)n, dp.wq.get(), dp.wk.get(),
                                                       dp.wv.get(), dp.wo.get(),
                                                       cfg_.k > 0.0 ? dp.ws.template as<double>() : nullptr,
                                                       df.template as<double>(), dy.get(), nullptr));
        } else {
            detail::check(skb_xcache_forward_chunk(h_.get(), dx.get(), (int64_t)n, dp.wq.get(), dp.wk.get(),
                                                   dp.wv.get(), dp.wo.get(),
                                                   cfg_.k > 0.0 ? dp.ws.template as<double>() : nullptr, dy.get(),
                                                   nullptr));
        }
        y.data = dy.to_host<T>(y.data.size());
        return y;
    }

    std::size_t capacity() const { return cap_; }
    std::size_t size() const { return state().sel; }
    std::size_t window_fill() const { return std::min<std::size_t>(positions_seen(), cfg_.window); }
    std::size_t positions_seen() const { return state().seen; }
    std::size_t peak_kv() const { return state().peak; }
    bool ever_evicted(std::size_t pos) const {
        std::vector<uint8_t> ev(pos + 1, 0);
        int64_t np = 0;
        detail::check(skb_cache_ledger(inner(), 0, 0, nullptr, 0, &np, ev.data(), (int64_t)ev.size(), nullptr, 0,
                                       nullptr));
        return ev[pos] != 0;
    }
    std::vector<std::size_t> drain_evictions() {
        int64_t np = 0;
        detail::check(skb_cache_ledger(inner(), 0, 0, nullptr, 0, &np, nullptr, 0, nullptr, 0, nullptr));
        std::vector<int64_t> pend((size_t)std::max<int64_t>(np, 1));
        detail::check(skb_cache_ledger(inner(), 0, 1, pend.data(), np, &np, nullptr, 0, nullptr, 0, nullptr));
        return std::vector<std::size_t>(pend.begin(), pend.begin() + np);
    }
    std::vector<std::size_t> retained_positions() const {
        const State s = state();
        std::vector<std::size_t> out(s.positions.begin(), s.positions.end());
        std::sort(out.begin(), out.end());
        return out;
    }
    double frozen_score(std::size_t pos) const {
        const std::size_t seen = positions_seen();
        if (pos >= seen) throw std::out_of_range("frozen_score: position not seen");
        std::vector<double> sc(pos + 1);
        int64_t np = 0;
        detail::check(skb_cache_ledger(inner(), 0, 0, nullptr, 0, &np, nullptr, 0, sc.data(), (int64_t)sc.size(),
                                       nullptr));
        return sc[pos];
    }
    // A snapshot of the cache's stream (StreamState through its wire format).
    const StreamState& stream() const {
        if (!(cfg_.k > 0.0)) throw ArgumentError("cache: no selection stream (k = 0)");
        std::vector<std::uint8_t> payload;
        serialize(payload);
        stream_snapshot_ = std::make_shared<StreamState>(stream_from_payload(payload));
        return *stream_snapshot_;
    }

    void serialize(std::vector<std::uint8_t>& out) const {  // cache.cpp:416-475 (the reference's payload)
        std::vector<double> ns(3);
        detail::check(skb_xcache_norm_state(h_.get(), ns.data(), 0, nullptr));
        size_t n = 0;
        detail::check(skb_cache_snapshot(inner(), 0, ns.data(), nullptr, &n, nullptr));
        std::vector<std::uint8_t> b(n);
        detail::check(skb_cache_snapshot(inner(), 0, ns.data(), b.data(), &n, nullptr));
        out.insert(out.end(), b.begin(), b.begin() + n);
    }
    static SparseKvCache deserialize(const std::uint8_t* data, std::size_t len, const AttnConfig& cfg,
                                     std::size_t d_model, const ScoringParams& scoring) {
        SparseKvCache c(cfg, d_model, scoring);
        std::vector<double> ns(3);
        detail::check(skb_cache_restore(c.inner(), 0, data, len, ns.data(), nullptr));
        detail::check(skb_xcache_norm_state(c.h_.get(), ns.data(), 1, nullptr));
        return c;
    }

    skb_xcache* handle() const { return h_.get(); }

  private:
    struct State {
        std::vector<int32_t> positions;
        std::size_t sel = 0, seen = 0, peak = 0;
        double tau = kNegInf;
    };
    skb_cache* inner() const { return skb_xcache_inner(h_.get()); }
    State state() const {
        State s;
        s.positions.resize(cap_ + cfg_.window + 2);
        int64_t cnt = 0, seen = 0, peak = 0;
        detail::check(skb_cache_state(inner(), 0, s.positions.data(), &cnt, &s.tau, &seen, &peak, nullptr));
        s.positions.resize((size_t)cnt);
        s.seen = (size_t)seen;
        s.peak = (size_t)peak;
        const std::size_t win = std::min<std::size_t>(s.seen, cfg_.window);
        s.sel = (size_t)cnt - std::min<std::size_t>((size_t)cnt, win);
        return s;
    }
    // the stream blob inside a cache payload (cache.cpp:416-475 field order)
    static StreamState stream_from_payload(const std::vector<std::uint8_t>& p) {
        size_t off = 0;
        auto u64 = [&]() {
            uint64_t v = 0;
            std::memcpy(&v, p.data() + off, 8);
            off += 8;
            return v;
        };
        off += 4 * 8 + 8 + 2;     // d_model, heads, window, cap, k, mode, has_stream
        const uint64_t t = u64();  // positions
        off += 8 + t * 8;          // score count + scores
        off += 8 * 4;              // norm state
        const uint64_t blen = u64();
        return StreamState::deserialize(p.data() + off, (size_t)blen, nullptr);
    }

    AttnConfig cfg_;
    std::size_t d_model_;
    ScoringParams scoring_;
    std::size_t max_pos_;
    std::size_t cap_ = 0;
    std::shared_ptr<skb_xcache> h_;
    mutable std::shared_ptr<StreamState> stream_snapshot_;
};

// Algorithm 3 (cache.cpp:548-563). Without a tape: the recurrence itself,
// chunk by chunk through one SparseKvCache. With a tape (training): the
// batch kernels over the whole sequence with stop-gradients at the chunk
// starts (attention.cpp:228-234) — the same outputs.
template <class T>
MatT<T> chunked_forward(const MatT<T>& x, std::size_t chunk_len, const AttnParams<T>& params,
                        const ScoringParams& scoring, const AttnConfig& cfg, AttnTape<T>* tape = nullptr,
                        const LinearMixParams<T>* lin = nullptr) {
    if (chunk_len == 0) throw ArgumentError("chunked_forward: chunk_len must be positive");
    if (lin || cfg.linear_mix) {  // Appendix B.1: the batch kernels, stop-gradients at the chunk starts
        if (!lin) throw ConfigError("forward_chunk: linear mix needs feature parameters");
        AttnConfig c = cfg;
        c.linear_mix = true;
        return detail::run_forward(x, params, scoring, c, tape, chunk_len, lin);
    }
    if (tape) return detail::run_forward(x, params, scoring, cfg, tape, chunk_len);
    SparseKvCache<T> cache(cfg, x.cols, scoring, std::max<std::size_t>(x.rows, 1));
    MatT<T> out(x.rows, x.cols);
    for (std::size_t base = 0; base < x.rows; base += chunk_len) {
        const std::size_t n = std::min(chunk_len, x.rows - base);
        MatT<T> chunk(n, x.cols);
        std::copy(x.row(base), x.row(base) + n * x.cols, chunk.data.begin());
        const MatT<T> y = cache.forward_chunk(chunk, params);
        std::copy(y.data.begin(), y.data.end(), out.row(base));
    }
    return out;
}

template <class T>
std::vector<std::size_t> prune_cache(SparseKvCache<T>& cache) {
    return cache.drain_evictions();
}

template <class T>
std::vector<T> generate_step(SparseKvCache<T>& cache, const std::vector<T>& new_token_state,
                             const AttnParams<T>& params, const LinearMixParams<T>* lin = nullptr) {
    MatT<T> x(1, new_token_state.size());
    std::copy(new_token_state.begin(), new_token_state.end(), x.data.begin());
    return cache.forward_chunk(x, params, nullptr, lin).data;
}

template <class T>
void save_cache_snapshot(const SparseKvCache<T>& cache, const std::string& path) {  // cache.cpp:579-595
    std::vector<std::uint8_t> payload;
    cache.serialize(payload);
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open for writing: " + path);
    f.write("SPKC", 4);
    const std::uint16_t ver = 1;
    f.put(static_cast<char>(ver & 0xff));
    f.put(static_cast<char>(ver >> 8));
    for (int i = 0; i < 8; ++i) f.put(static_cast<char>((payload.size() >> (8 * i)) & 0xff));
    f.write(reinterpret_cast<const char*>(payload.data()), static_cast<std::streamsize>(payload.size()));
    if (!f) throw IoError("write failed: " + path);
}

template <class T>
SparseKvCache<T> load_cache_snapshot(const std::string& path, const AttnConfig& cfg, std::size_t d_model,
                                     const ScoringParams& scoring) {  // cache.cpp:597-618
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open: " + path);
    char magic[4];
    f.read(magic, 4);
    if (!f || std::memcmp(magic, "SPKC", 4) != 0) throw IoError("not a cache snapshot: " + path);
    const int lo = f.get(), hi = f.get();
    if (lo < 0 || hi < 0) throw IoError("cache snapshot: truncated header");
    if ((lo | (hi << 8)) != 1) throw IoError("cache snapshot: unsupported version");
    std::uint8_t lenb[8];
    f.read(reinterpret_cast<char*>(lenb), 8);
    if (!f) throw IoError("cache snapshot: truncated header");
    std::uint64_t plen = 0;
    for (int i = 0; i < 8; ++i) plen |= static_cast<std::uint64_t>(lenb[i]) << (8 * i);
    std::vector<std::uint8_t> payload(plen);
    f.read(reinterpret_cast<char*>(payload.data()), static_cast<std::streamsize>(plen));
    if (!f) throw IoError("cache snapshot: truncated payload");
    return SparseKvCache<T>::deserialize(payload.data(), payload.size(), cfg, d_model, scoring);
}

}  // namespace sparsek
