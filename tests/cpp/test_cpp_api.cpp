// C++ drop-in surface (include/sparsek_b200.hpp) over libsparsek_b200.so.
//   ./test_cpp_api cpu  -> error mapping that needs no device (config validation)
//   ./test_cpp_api gpu  -> operator / stream / attention values on a B200
// Values follow the reference's own examples: sparsek([0.9,0.5,0.1], 2) ->
// p = [1, 0.7, 0.3], tau = -0.2 (proj/tests/test_sparsek_op.cpp:131-144), and
// the dense limit of the attention (proj/tests/test_attention.cpp:13-42).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "sparsek_b200.hpp"

using namespace sparsek_b200;

#define EXPECT(c)                                                    \
    do {                                                             \
        if (!(c)) {                                                  \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                \
        }                                                            \
    } while (0)

template <class E, class F>
bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static int cpu_checks() {
    AttnConfig bad;
    bad.k = -1.0;
    EXPECT(throws<ConfigError>([&] { SparseKAttention a(1, 16, 8, bad, DType::f32); }));
    AttnConfig none;
    none.k = 0.5;
    none.window = 0;
    EXPECT(throws<ConfigError>([&] { SparseKAttention a(1, 16, 8, none, DType::f32); }));
    EXPECT(throws<ArgumentError>([&] { sparsek({}, 2.0); }));
    EXPECT(throws<ArgumentError>([&] { sparsek({1.0}, -2.0); }));
    EXPECT(throws<NumericError>([&] { sparsek({1.0, NAN}, 1.0); }));
    std::printf("cpu ok\n");
    return 0;
}

static int gpu_checks() {
    const SparseKSolution s = sparsek({0.9, 0.5, 0.1}, 2.0);
    EXPECT(std::fabs(s.p[0] - 1.0) < 1e-12 && std::fabs(s.p[1] - 0.7) < 1e-12 && std::fabs(s.p[2] - 0.3) < 1e-12);
    EXPECT(std::fabs(s.tau + 0.2) < 1e-12 && s.u_count == 1 && s.w_count == 3);
    const auto j = sparsek_jvp({0.9, 0.5, 0.1}, 2.0, {0.0, 4.0, 2.0});
    EXPECT(std::fabs(j[0]) < 1e-12 && std::fabs(j[1] - 1.0) < 1e-12 && std::fabs(j[2] + 1.0) < 1e-12);
    // stream == batch solve on every prefix
    StreamState st(3.0);
    std::vector<double> z = {0.3, -1.2, 2.5, 0.7, 0.1, 1.9, -0.4, 0.8, 1.1, -2.0, 0.5, 0.6};
    for (size_t t = 0; t < z.size(); ++t) {
        const auto r = st.push(z[t]);
        std::vector<double> pre(z.begin(), z.begin() + t + 1);
        const auto b = sparsek(pre, 3.0);
        if (!b.infeasible && !b.degenerate) EXPECT(std::fabs(r.tau - b.tau) < 1e-12);
    }
    // attention: budget covering every position == dense causal softmax attention
    const int B = 1, L = 48, H = 2, P = 16;
    AttnConfig cfg;
    cfg.k = 1000.0;
    cfg.window = 3;
    cfg.heads = H;
    std::vector<float> q(B * L * H * P), k(q.size()), v(q.size()), o(q.size());
    std::vector<double> u(B * L);
    unsigned seed = 7;
    auto rnd = [&] {
        seed = seed * 1664525u + 1013904223u;
        return ((seed >> 8) & 0xFFFF) / 32768.0f - 1.0f;
    };
    for (auto* vec : {&q, &k, &v})
        for (auto& x : *vec) x = rnd();
    for (auto& x : u) x = rnd();
    DeviceBuffer dq(q.size() * 4), dk(q.size() * 4), dv(q.size() * 4), dout(q.size() * 4), du(u.size() * 8),
        dlse((size_t)B * H * L * 8);
    cuda_check(cudaMemcpy(dq.get(), q.data(), q.size() * 4, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(dk.get(), k.data(), q.size() * 4, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(dv.get(), v.data(), q.size() * 4, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(du.get(), u.data(), u.size() * 8, cudaMemcpyHostToDevice), "H2D");
    SparseKAttention attn(B, L, P, cfg, DType::f32);
    attn.forward(dq.get(), dk.get(), dv.get(), (const double*)du.get(), dout.get(), (double*)dlse.get());
    cuda_check(cudaMemcpy(o.data(), dout.get(), o.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    double maxerr = 0.0;
    const double scale = 1.0 / std::sqrt((double)P);
    for (int i = 0; i < L; ++i)
        for (int h = 0; h < H; ++h) {
            std::vector<double> a(i + 1);
            double mx = -1e300, den = 0.0;
            for (int j2 = 0; j2 <= i; ++j2) {
                double d = 0;
                for (int c = 0; c < P; ++c) d += (double)q[(i * H + h) * P + c] * k[(j2 * H + h) * P + c];
                a[j2] = d * scale;
                mx = std::max(mx, a[j2]);
            }
            for (int j2 = 0; j2 <= i; ++j2) den += (a[j2] = std::exp(a[j2] - mx));
            for (int c = 0; c < P; ++c) {
                double acc = 0;
                for (int j2 = 0; j2 <= i; ++j2) acc += a[j2] / den * v[(j2 * H + h) * P + c];
                maxerr = std::max(maxerr, std::fabs(acc - (double)o[(i * H + h) * P + c]));
            }
        }
    EXPECT(maxerr < 1e-5);
    // incremental scoring: 1 + 5 + 10 rows through ScoreState == one 16-row call (bit for bit)
    {
        const int SB = 2, SN = 16, SD = 8;
        std::vector<double> x(SB * SN * SD), w(SD);
        for (auto& e : x) e = rnd();
        for (auto& e : w) e = rnd();
        DeviceBuffer dx(x.size() * 8), dw(w.size() * 8), r1(SB * SN * 8), u1(SB * SN * 8), r2(SB * SN * 8),
            u2(SB * SN * 8);
        cuda_check(cudaMemcpy(dw.get(), w.data(), w.size() * 8, cudaMemcpyHostToDevice), "H2D");
        ScoringConfig sc;
        ScoreState one(SB, SD, sc), parts(SB, SD, sc);
        cuda_check(cudaMemcpy(dx.get(), x.data(), x.size() * 8, cudaMemcpyHostToDevice), "H2D");
        one.score(dx.get(), DType::f64, SN, (const double*)dw.get(), (double*)r1.get(), (double*)u1.get());
        std::vector<double> ua(SB * SN), ub(SB * SN);
        cuda_check(cudaMemcpy(ua.data(), u1.get(), ua.size() * 8, cudaMemcpyDeviceToHost), "D2H");
        int off = 0;
        for (int n : {1, 5, 10}) {  // rows [off, off + n) of every sequence, packed [B, n, D]
            std::vector<double> xs(SB * n * SD);
            for (int b2 = 0; b2 < SB; ++b2)
                for (int i = 0; i < n * SD; ++i) xs[(b2 * n) * SD + i] = x[(b2 * SN + off) * SD + i];
            DeviceBuffer dxs(xs.size() * 8), rs(SB * n * 8), us(SB * n * 8);
            cuda_check(cudaMemcpy(dxs.get(), xs.data(), xs.size() * 8, cudaMemcpyHostToDevice), "H2D");
            parts.score(dxs.get(), DType::f64, n, (const double*)dw.get(), (double*)rs.get(), (double*)us.get());
            std::vector<double> uh(SB * n);
            cuda_check(cudaMemcpy(uh.data(), us.get(), uh.size() * 8, cudaMemcpyDeviceToHost), "D2H");
            for (int b2 = 0; b2 < SB; ++b2)
                for (int i = 0; i < n; ++i) ub[b2 * SN + off + i] = uh[b2 * n + i];
            off += n;
        }
        for (int i = 0; i < SB * SN; ++i) EXPECT(ua[i] == ub[i]);
    }
    // cache snapshot round trip: a restored cache continues bit-identically
    {
        const int CL = 64, CH = 2, CP = 32;
        AttnConfig cc;
        cc.k = 6.5;
        cc.window = 5;
        cc.heads = CH;
        SparseKvCache a(1, CL, CP, cc, DType::f32), b2(1, CL, CP, cc, DType::f32);
        std::vector<float> row(CH * CP);
        DeviceBuffer dq2(row.size() * 4), dk2(row.size() * 4), dv2(row.size() * 4), du2(8), do1(row.size() * 4),
            do2(row.size() * 4);
        auto feed = [&](SparseKvCache& c, int i, void* o) {
            seed = 1234u + 7u * (unsigned)i;
            for (auto& e : row) e = rnd();
            cuda_check(cudaMemcpy(dq2.get(), row.data(), row.size() * 4, cudaMemcpyHostToDevice), "H2D");
            for (auto& e : row) e = rnd();
            cuda_check(cudaMemcpy(dk2.get(), row.data(), row.size() * 4, cudaMemcpyHostToDevice), "H2D");
            for (auto& e : row) e = rnd();
            cuda_check(cudaMemcpy(dv2.get(), row.data(), row.size() * 4, cudaMemcpyHostToDevice), "H2D");
            const double uu = rnd() + 0.01 * i;
            cuda_check(cudaMemcpy(du2.get(), &uu, 8, cudaMemcpyHostToDevice), "H2D");
            c.step(dq2.get(), dk2.get(), dv2.get(), (const double*)du2.get(), o);
        };
        for (int i = 0; i < 40; ++i) feed(a, i, do1.get());
        b2.deserialize(0, a.serialize(0));
        std::vector<float> o1(row.size()), o2(row.size());
        for (int i = 40; i < CL; ++i) {
            feed(a, i, do1.get());
            feed(b2, i, do2.get());
            cuda_check(cudaMemcpy(o1.data(), do1.get(), o1.size() * 4, cudaMemcpyDeviceToHost), "D2H");
            cuda_check(cudaMemcpy(o2.data(), do2.get(), o2.size() * 4, cudaMemcpyDeviceToHost), "D2H");
            EXPECT(std::memcmp(o1.data(), o2.data(), o1.size() * 4) == 0);
        }
        EXPECT(a.serialize(0) == b2.serialize(0));
    }
    std::printf("gpu ok (dense-limit max err %.3g)\n", maxerr);
    return 0;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    try {
        return gpu ? gpu_checks() : cpu_checks();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 2;
    }
}
