// K1 — the KV scoring network u_j = w . x_j, its timestep normalisation and
// position slope (proj/include/sparsek/selection.hpp:69-96, Welford
// proj/src/selection.cpp:13-20), and its backward (proj/src/attention.cpp:
// 482-516 and the dx term at :564).
//
// Forward arithmetic is the reference's, operation for operation: raw is a
// sequential float64 dot product with separate multiply and add (the
// reference's x86-64 build has no FMA contraction), and the Welford recurrence
// runs in order per sequence with correctly rounded div/sqrt, so u is
// bit-identical to the reference's for identical x rows and w. Backward turns
// the reference's O(L^2) pullback into three suffix sums.
#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

namespace {

template <class S>
__device__ __forceinline__ double ldd(const S* p, int64_t i) {
    return (double)p[i];
}
template <>
__device__ __forceinline__ double ldd<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
    return (double)__bfloat162float(p[i]);
}

// One thread per row: raw = sum_c x[c] * w[c], left to right, no FMA.
// (Fallback for rows that are not 16-byte aligned.)
template <class S>
__global__ void k_score_raw(const S* __restrict__ x, const double* __restrict__ w, int64_t rows,
                            int D, double* __restrict__ raw) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const S* xr = x + r * D;
    double acc = 0.0;
    for (int c = 0; c < D; ++c) acc = __dadd_rn(acc, __dmul_rn(ldd<S>(xr, c), w[c]));
    raw[r] = acc;
}

// The same dot products, HBM-streamed: a CTA owns 128 rows; the rows are
// staged through shared memory in 128-byte column slices (a 4-deep cp.async
// ring, 8 threads per row so each row's slice is one coalesced 128-byte
// read), and thread r then walks its row's slice in column order — the
// reference's left-to-right, unfused float64 accumulation, so raw stays
// bit-identical (proj/include/sparsek/selection.hpp:72-74).
#ifndef SKB_K1_ROWS
#define SKB_K1_ROWS 32  // cfg3 x: 62.5 us vs 76.7 at 128 rows (more CTAs, shorter staging)
#endif
constexpr int kRawRows = SKB_K1_ROWS;  // rows (threads) per CTA
constexpr int kRawStages = 4;
constexpr int kRawPitch = 144;  // 128 B slice + 16 B pad: 16-byte row reads spread over the banks

template <class S>
__global__ void __launch_bounds__(kRawRows) k_score_raw_tiled(const S* __restrict__ x, const double* __restrict__ w,
                                                              int64_t rows, int D, double* __restrict__ raw) {
    constexpr int kCols = 128 / (int)sizeof(S);  // columns per 128-byte slice
    constexpr int kVec = 16 / (int)sizeof(S);    // columns per 16-byte chunk
    constexpr int kStageB = kRawRows * kRawPitch + kCols * 8;  // x slice rows, then the w slice (float64)
    extern __shared__ __align__(16) uint8_t raw_smem[];
    auto tile = [&](int st) { return raw_smem + st * kStageB; };
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * kRawRows;
    const int nslices = (D + kCols - 1) / kCols;
    auto cp16 = [](uint8_t* dst, const void* src, bool ok) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
    };
    auto issue = [&](int sl) {
        uint8_t* dst = tile(sl % kRawStages);
        const int c0 = sl * kCols;
#pragma unroll
        for (int it = 0; it < 8; ++it) {  // 128 rows x 8 chunks / 128 threads
            const int idx = it * kRawRows + t;
            const int rr = idx >> 3, ch = idx & 7;
            const int64_t row = r0 + rr;
            const int c = c0 + ch * kVec;
            const bool ok = row < rows && c < D;
            cp16(dst + rr * kRawPitch + ch * 16, x + (ok ? row * D + c : 0), ok);
        }
        if (t < kCols / 2) {  // w[c0 .. c0 + kCols) as float64 pairs
            const int c = c0 + 2 * t;
            cp16(dst + kRawRows * kRawPitch + t * 16, w + (c < D ? c : 0), c + 1 < D);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int sl = 0; sl < kRawStages - 1; ++sl) {
        if (sl < nslices) issue(sl);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    double acc = 0.0;
    for (int sl = 0; sl < nslices; ++sl) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kRawStages - 2) : "memory");
        __syncthreads();  // slice sl landed for every thread; slot (sl-1) % stages is free
        if (sl + kRawStages - 1 < nslices) issue(sl + kRawStages - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        const uint8_t* rowp = tile(sl % kRawStages) + t * kRawPitch;
        const double* ws = reinterpret_cast<const double*>(tile(sl % kRawStages) + kRawRows * kRawPitch);
        const int c0 = sl * kCols;
        if (c0 + kCols <= D) {  // a full slice: no per-element predicate
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                const uint4 v = *reinterpret_cast<const uint4*>(rowp + ch * 16);
                const S* e = reinterpret_cast<const S*>(&v);
                double prod[kVec];
#pragma unroll
                for (int q = 0; q < kVec; ++q) prod[q] = __dmul_rn(ldd<S>(e, q), ws[ch * kVec + q]);
#pragma unroll
                for (int q = 0; q < kVec; ++q) acc = __dadd_rn(acc, prod[q]);
            }
        } else {
            const int n = D - c0;
            for (int c = 0; c < n; ++c) {
                const S* e = reinterpret_cast<const S*>(rowp);
                acc = __dadd_rn(acc, __dmul_rn(ldd<S>(e, c), __ldg(w + c0 + c)));
            }
        }
    }
    if (r0 + t < rows) raw[r0 + t] = acc;
}

// Correctly rounded a / n for a positive integer count n, given y = RN(1/n):
// q0 = RN(a y) is within an ulp of a/n, the residual a - q0 n is exact in
// one fma, and RN(q0 + r y) is then RN(a/n) (Markstein's theorem) — the same
// value as __ddiv_rn, with the reciprocal off the dependency chain. (A zero
// dividend gives +0; the callers' dividends are never -0: raw sums start at
// +0.0, so rin - mu and m2 cannot be negative zeros.)
__device__ __forceinline__ double div_by_count(double a, double n, double y) {
    const double q0 = __dmul_rn(a, y);
    return __fma_rn(__fma_rn(-q0, n, a), y, q0);
}

// Sequential Welford per sequence; emits the statistics the parallel finish
// needs. The mean recurrence is a serial float64 chain (bit-identity with the
// reference forbids reassociation), so one thread runs it — on operands
// staged in shared memory by a second warp, which also computes the
// reciprocals 1/(i+1) off the chain and writes the previous block's results
// out coalesced. Per step the chain is sub, mul, two fmas and an add.
constexpr int kWfBlock = 256;

__global__ void __launch_bounds__(64) k_score_welford(const double* __restrict__ raw, int L, skb_scoring sc,
                                                      double* __restrict__ mean, double* __restrict__ var,
                                                      int* __restrict__ bad, const int* ready) {
    __shared__ double s_rin[2][kWfBlock], s_y[2][kWfBlock], s_mu[2][kWfBlock], s_v[2][kWfBlock];
    const int b = blockIdx.x;
    const double* rb = raw + (int64_t)b * L;
    double* mb = mean + (int64_t)b * L;
    double* vb = var + (int64_t)b * L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (L + kWfBlock - 1) / kWfBlock;
    bool nonfinite = false;
    auto prep = [&](int k) {
        const int buf = k & 1;
        if (ready) {  // streaming: wait until the producer has stored these rows (128-row blocks of B*L)
            const int64_t r0 = (int64_t)b * L + (int64_t)k * kWfBlock;
            const int64_t r1 = (int64_t)b * L + min(L, (k + 1) * kWfBlock) - 1;
            for (int64_t blk = r0 / 128 + lane; blk <= r1 / 128; blk += 32) {
                int f = 0;
                while (true) {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(ready + blk) : "memory");
                    if (f) break;
                    __nanosleep(256);
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int e = 0; e < kWfBlock / 32; ++e) {
            const int j = e * 32 + lane;
            const int i = k * kWfBlock + j;
            const double r = i < L ? rb[i] : 0.0;
            nonfinite |= !isfinite(r);
            const double slope = sc.slope_enabled ? __dmul_rn((double)(i + 1), sc.slope_eps) : 0.0;
            s_rin[buf][j] = sc.slope_order == 0 ? __dadd_rn(r, slope) : r;
            s_y[buf][j] = __drcp_rn((double)(i + 1));
        }
    };
    auto flush = [&](int k) {
        const int buf = k & 1;
        for (int j = lane; j < kWfBlock; j += 32) {
            const int i = k * kWfBlock + j;
            if (i < L) {
                mb[i] = s_mu[buf][j];
                vb[i] = s_v[buf][j];
            }
        }
    };
    if (warp == 1) prep(0);
    __syncthreads();
    double mu = 0.0, m2 = 0.0;
    for (int k = 0; k < nblk; ++k) {
        const int buf = k & 1;
        if (threadIdx.x == 0) {
            const int n = min(kWfBlock, L - k * kWfBlock);
            const double* rin_s = s_rin[buf];
            const double* y_s = s_y[buf];
#pragma unroll 4
            for (int j = 0; j < n; ++j) {
                const double rin = rin_s[j], y = y_s[j];
                const double cnt = (double)(k * kWfBlock + j + 1);
                const double delta = __dsub_rn(rin, mu);
                mu = __dadd_rn(mu, div_by_count(delta, cnt, y));
                m2 = __dadd_rn(m2, __dmul_rn(delta, __dsub_rn(rin, mu)));
                s_mu[buf][j] = mu;
                s_v[buf][j] = div_by_count(m2, cnt, y);
            }
        } else if (warp == 1) {
            if (k + 1 < nblk) prep(k + 1);
            if (k >= 1) flush(k - 1);
        }
        __syncthreads();
    }
    if (warp == 1) flush(nblk - 1);
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0 && warp == 1) *bad = 1;
}

// Incremental scoring for decoding (score_tokens with base_pos, TimestepNormState
// carried across calls; proj/src/selection.cpp:13-31): n new rows per sequence
// continue the Welford state [count, mean, m2] exactly as the reference's
// push does, operation for operation.
// (rawv and raw_out may alias: the continuation rewrites raw in place)
__global__ void k_score_continue(const double* rawv, int n, skb_scoring sc, double* __restrict__ state,
                                 double* raw_out, double* __restrict__ u_out, int* __restrict__ bad) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= gridDim.x * blockDim.x) return;
    double* stt = state + (int64_t)b * 3;
    double cnt = stt[0], mu = stt[1], m2 = stt[2];
    for (int i = 0; i < n; ++i) {
        const int64_t r = (int64_t)b * n + i;
        const double rw = rawv[r];
        if (!isfinite(rw)) *bad = 1;
        const double slope = sc.slope_enabled ? __dmul_rn(__dadd_rn(cnt, 1.0), sc.slope_eps) : 0.0;
        if (sc.norm_mode == 0) {
            raw_out[r] = rw;
            u_out[r] = __dadd_rn(rw, slope);
            cnt = __dadd_rn(cnt, 1.0);
            continue;
        }
        const double rin = sc.slope_order == 0 ? __dadd_rn(rw, slope) : rw;
        cnt = __dadd_rn(cnt, 1.0);
        const double delta = __dsub_rn(rin, mu);
        mu = __dadd_rn(mu, __ddiv_rn(delta, cnt));
        m2 = __dadd_rn(m2, __dmul_rn(delta, __dsub_rn(rin, mu)));
        const double sd = __dsqrt_rn(__dadd_rn(__ddiv_rn(m2, cnt), 1e-5));
        const double z = __ddiv_rn(__dsub_rn(rin, mu), sd);
        raw_out[r] = rin;
        u_out[r] = sc.slope_order == 0 ? z : __dadd_rn(z, slope);
    }
    stt[0] = cnt;
    stt[1] = mu;
    stt[2] = m2;
}

// (raw_in and raw may alias: the caller stages the dot products in raw)
__global__ void k_score_finish(const double* raw_in, int64_t n, int L, skb_scoring sc, double* raw,
                               double* __restrict__ u,
                               double* __restrict__ mean, double* __restrict__ sdev_var,
                               int* __restrict__ bad) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int i = (int)(r % L);
    const double rw = raw_in[r];
    if (!isfinite(rw)) *bad = 1;
    const double slope = sc.slope_enabled ? __dmul_rn((double)(i + 1), sc.slope_eps) : 0.0;
    if (sc.norm_mode == 0) {
        raw[r] = rw;
        u[r] = __dadd_rn(rw, slope);
        mean[r] = 0.0;
        sdev_var[r] = 1.0;
        return;
    }
    const double rin = sc.slope_order == 0 ? __dadd_rn(rw, slope) : rw;
    const double mu = mean[r];
    const double sd = __dsqrt_rn(__dadd_rn(sdev_var[r], 1e-5));
    const double z = __ddiv_rn(__dsub_rn(rin, mu), sd);
    raw[r] = rin;
    u[r] = sc.slope_order == 0 ? z : __dadd_rn(z, slope);
    sdev_var[r] = sd;
}

// ---------------------------------------------------------------- backward
// Suffix sums of A = coef/(j+1), Bc = coef*y/((j+1)s), Cc = Bc*mu, coef = gu/s.
__global__ void __launch_bounds__(1024)
k_score_pullback(const double* __restrict__ gu, const double* __restrict__ raw,
                 const double* __restrict__ mean, const double* __restrict__ sdev, int L,
                 int norm_mode, double* __restrict__ graw) {
    __shared__ double w3[3][32];
    const int b = blockIdx.x;
    const int64_t bl = (int64_t)b * L;
    if (norm_mode == 0) {
        for (int j = threadIdx.x; j < L; j += blockDim.x) graw[bl + j] = gu[bl + j];
        return;
    }
    const int per = (L + blockDim.x - 1) / blockDim.x;
    // reversed order: thread 0 owns the tail so an inclusive scan gives suffix sums
    const int hi = L - min(L, (int)threadIdx.x * per);
    const int lo = max(0, hi - per);
    auto terms = [&](int j, double& A, double& Bc, double& Cc) {
        const double g = gu[bl + j];
        const double s = sdev[bl + j], mu = mean[bl + j];
        const double cnt = (double)(j + 1);
        const double coef = g / s;
        const double y = (raw[bl + j] - mu) / s;
        A = coef / cnt;
        Bc = coef * y / (cnt * s);
        Cc = Bc * mu;
    };
    double sA = 0.0, sB = 0.0, sC = 0.0;
    for (int j = lo; j < hi; ++j) {
        double A, Bc, Cc;
        terms(j, A, Bc, Cc);
        sA += A;
        sB += Bc;
        sC += Cc;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double iA = sA, iB = sB, iC = sC;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double a = __shfl_up_sync(0xffffffffu, iA, o);
        const double bb = __shfl_up_sync(0xffffffffu, iB, o);
        const double c = __shfl_up_sync(0xffffffffu, iC, o);
        if (lane >= o) {
            iA += a;
            iB += bb;
            iC += c;
        }
    }
    if (lane == 31) {
        w3[0][wid] = iA;
        w3[1][wid] = iB;
        w3[2][wid] = iC;
    }
    __syncthreads();
    double pA = 0.0, pB = 0.0, pC = 0.0;
    for (int w = 0; w < wid; ++w) {
        pA += w3[0][w];
        pB += w3[1][w];
        pC += w3[2][w];
    }
    // suffix sums strictly after this thread's range
    double rA = pA + iA - sA, rB = pB + iB - sB, rC = pC + iC - sC;
    for (int j = hi - 1; j >= lo; --j) {
        double A, Bc, Cc;
        terms(j, A, Bc, Cc);
        rA += A;
        rB += Bc;
        rC += Cc;
        const double coef = gu[bl + j] / sdev[bl + j];
        graw[bl + j] = coef - rA - raw[bl + j] * rB + rC;
    }
}

// Chunk-wise training: graw[j2] only collects from j >= j2 in j2's own chunk
// (proj/src/attention.cpp:491, `for j2 = cs_of[j] ..`): one thread per
// (sequence, chunk) runs the suffix sums backwards over its chunk.
__global__ void k_score_pullback_chunked(const double* __restrict__ gu, const double* __restrict__ raw,
                                         const double* __restrict__ mean, const double* __restrict__ sdev, int L,
                                         int chunk_len, int nchunks, double* __restrict__ graw) {
    const int b = blockIdx.y;
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= nchunks) return;
    const int64_t bl = (int64_t)b * L;
    const int lo = ch * chunk_len, hi = min(L, lo + chunk_len);
    double rA = 0.0, rB = 0.0, rC = 0.0;
    for (int j = hi - 1; j >= lo; --j) {
        const double g = gu[bl + j];
        const double s = sdev[bl + j], mu = mean[bl + j];
        const double cnt = (double)(j + 1);
        const double coef = g / s;
        const double y = (raw[bl + j] - mu) / s;
        rA += coef / cnt;
        rB += coef * y / (cnt * s);
        rC += coef * y / (cnt * s) * mu;
        graw[bl + j] = coef - rA - raw[bl + j] * rB + rC;
    }
}

// dw_score[c] = sum_{b,j} graw[b,j] * x[b,j,c]: column blocks x row slabs, atomics across slabs.
template <class S>
__global__ void k_dw_score(const S* __restrict__ x, const double* __restrict__ graw, int64_t rows,
                           int D, int rows_per, double* __restrict__ dw) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= D) return;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per;
    const int64_t r1 = min(rows, r0 + rows_per);
    double acc = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
        const double g = graw[r];
        if (g != 0.0) acc += g * ldd<S>(x, r * D + c);
    }
    atomicAdd(dw + c, acc);
}

template <class S>
__global__ void k_dx_add(S* __restrict__ dx, const double* __restrict__ graw,
                         const double* __restrict__ w, int64_t rows, int D) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * D) return;
    const int64_t r = i / D;
    const int c = (int)(i % D);
    dx[i] = (S)((double)dx[i] + graw[r] * w[c]);
}
template <>
__global__ void k_dx_add<__nv_bfloat16>(__nv_bfloat16* __restrict__ dx, const double* __restrict__ graw,
                                        const double* __restrict__ w, int64_t rows, int D) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * D) return;
    const int64_t r = i / D;
    const int c = (int)(i % D);
    dx[i] = __float2bfloat16((float)((double)__bfloat162float(dx[i]) + graw[r] * w[c]));
}

template <class F>
void dispatch_x(int32_t dt, F&& f) {
    if (dt == SKB_F64) f((const double*)nullptr);
    else if (dt == SKB_F32) f((const float*)nullptr);
    else if (dt == SKB_BF16) f((const __nv_bfloat16*)nullptr);
    else throw Error(SKB_EARG, "score: unsupported x dtype");
}

// raw[r] = x[r, :] . w for rows r: the staged kernel when rows are 16-byte
// aligned, the row-per-thread kernel otherwise.
void launch_raw(int32_t xdt, const void* x, const double* w, int64_t rows, int64_t D, double* out, cudaStream_t st) {
    dispatch_x(xdt, [&](auto tag) {
        using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
        const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (D * (int64_t)sizeof(S)) % 16 == 0;
        constexpr int smem = kRawStages * (kRawRows * kRawPitch + (128 / (int)sizeof(S)) * 8);
        static uint64_t attr_set = 0;
        if (aligned && first_on_device(&attr_set))
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_score_raw_tiled<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                smem));
        if (aligned)
            k_score_raw_tiled<S><<<(unsigned)cdiv(rows, kRawRows), kRawRows, smem, st>>>(static_cast<const S*>(x),
                                                                                       w, rows, (int)D, out);
        else
            k_score_raw<S><<<(unsigned)cdiv(rows, 128), 128, 0, st>>>(static_cast<const S*>(x), w, rows, (int)D,
                                                                        out);
    });
}

// The non-finite-input flag: one persistent device word per (thread,
// device) and a pinned host word to read it back (no per-call allocation).
int* bad_flag() {
    thread_local int* flags[64] = {};
    int dev = 0;
    SKB_CHECK_CUDA(cudaGetDevice(&dev));
    int*& f = flags[dev & 63];
    if (!f) SKB_CHECK_CUDA(cudaMalloc(&f, sizeof(int)));
    return f;
}
bool read_flag(const int* bad, cudaStream_t st) {
    thread_local int* host = nullptr;
    if (!host) SKB_CHECK_CUDA(cudaMallocHost(&host, sizeof(int)));
    SKB_CHECK_CUDA(cudaMemcpyAsync(host, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    return *host != 0;
}

}  // namespace

void run_score_fwd(int64_t B, int64_t L, int64_t D, int32_t xdt, const void* x, const double* w,
                   const skb_scoring& sc, double* raw, double* u, double* mean, double* sdev,
                   cudaStream_t st) {
    SKB_REQUIRE(B >= 1 && L >= 1 && D >= 1, SKB_ESHAPE, "score_tokens: empty input");
    SKB_REQUIRE(sc.slope_eps > 0.0, SKB_EARG, "ScoringParams: slope_eps must be positive");
    const int64_t rows = B * L;
    int* bad = bad_flag();
    SKB_CHECK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    // raw is produced into `u` first (scratch), finished into raw/u below.
    launch_raw(xdt, x, w, rows, D, u, st);
    SKB_CHECK_LAUNCH();
    if (sc.norm_mode != 0) {
        k_score_welford<<<(unsigned)B, 64, 0, st>>>(u, (int)L, sc, mean, sdev, bad, nullptr);
        SKB_CHECK_LAUNCH();
    }
    // finish: reads raw from `u`; stage it in raw first
    SKB_CHECK_CUDA(cudaMemcpyAsync(raw, u, rows * sizeof(double), cudaMemcpyDeviceToDevice, st));
    k_score_finish<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(raw, rows, (int)L, sc, raw, u, mean,
                                                             sdev, bad);
    SKB_CHECK_LAUNCH();
    SKB_REQUIRE(!read_flag(bad, st), SKB_ENUMERIC, "score: non-finite value");
}

// Welford + finish on dot products already in `raw_in` (or arriving: `ready`
// non-null = per-128-row readiness flags set by the fused projection GEMM,
// skb_proj.cu); launches only, the caller checks *bad after synchronising.
void run_score_finish_async(int64_t B, int64_t L, const skb_scoring& sc, const double* raw_in, const int* ready,
                            double* raw, double* u, double* mean, double* sdev, int* bad, cudaStream_t st) {
    const int64_t rows = B * L;
    if (sc.norm_mode != 0) {
        k_score_welford<<<(unsigned)B, 64, 0, st>>>(raw_in, (int)L, sc, mean, sdev, bad, ready);
        SKB_CHECK_LAUNCH();
    }
    if (raw != raw_in)
        SKB_CHECK_CUDA(cudaMemcpyAsync(raw, raw_in, rows * sizeof(double), cudaMemcpyDeviceToDevice, st));
    k_score_finish<<<(unsigned)cdiv(rows, 256), 256, 0, st>>>(raw, rows, (int)L, sc, raw, u, mean, sdev, bad);
    SKB_CHECK_LAUNCH();
}
int* score_bad_flag() { return bad_flag(); }
bool score_read_flag(const int* bad, cudaStream_t st) { return read_flag(bad, st); }

void run_score_raw(int64_t rows, int64_t D, int32_t xdt, const void* x, const double* w, double* raw,
                   cudaStream_t st) {
    SKB_REQUIRE(rows >= 1 && D >= 1, SKB_ESHAPE, "score_tokens: empty input");
    launch_raw(xdt, x, w, rows, D, raw, st);
    SKB_CHECK_LAUNCH();
}

void run_score_continue(int64_t B, int64_t n, int64_t D, int32_t xdt, const void* x, const double* w,
                        const skb_scoring& sc, double* state, double* raw, double* u, cudaStream_t st) {
    SKB_REQUIRE(B >= 1 && n >= 1 && D >= 1, SKB_ESHAPE, "score_tokens: empty input");
    SKB_REQUIRE(sc.slope_eps > 0.0, SKB_EARG, "ScoringParams: slope_eps must be positive");
    const int64_t rows = B * n;
    int* bad = bad_flag();
    SKB_CHECK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    launch_raw(xdt, x, w, rows, D, raw, st);
    SKB_CHECK_LAUNCH();
    // raw holds the dot products; the continuation rewrites raw/u in place
    k_score_continue<<<(unsigned)B, 1, 0, st>>>(raw, (int)n, sc, state, raw, u, bad);
    SKB_CHECK_LAUNCH();
    SKB_REQUIRE(!read_flag(bad, st), SKB_ENUMERIC, "score: non-finite value");
}

void run_score_bwd(int64_t B, int64_t L, int64_t D, int32_t xdt, const void* x, const double* w,
                   const skb_scoring& sc, const double* gu, const double* raw, const double* mean,
                   const double* sdev, double* graw, double* dw, void* dx, cudaStream_t st) {
    const int64_t rows = B * L;
    SKB_REQUIRE(sc.chunk_len >= 0, SKB_EARG, "chunked_forward: chunk_len must be positive");
    if (sc.norm_mode != 0 && sc.chunk_len > 0 && sc.chunk_len < L) {
        const int nch = (int)cdiv(L, sc.chunk_len);
        k_score_pullback_chunked<<<dim3((unsigned)cdiv(nch, 128), (unsigned)B), 128, 0, st>>>(
            gu, raw, mean, sdev, (int)L, sc.chunk_len, nch, graw);
    } else {
        k_score_pullback<<<(unsigned)B, 1024, 0, st>>>(gu, raw, mean, sdev, (int)L, sc.norm_mode, graw);
    }
    SKB_CHECK_LAUNCH();
    if (dw) {
        SKB_CHECK_CUDA(cudaMemsetAsync(dw, 0, D * sizeof(double), st));
        const int rows_per = 256;
        dim3 g((unsigned)cdiv(D, 128), (unsigned)cdiv(rows, rows_per));
        dispatch_x(xdt, [&](auto tag) {
            using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
            k_dw_score<S><<<g, 128, 0, st>>>(static_cast<const S*>(x), graw, rows, (int)D, rows_per, dw);
        });
        SKB_CHECK_LAUNCH();
    }
    if (dx) {
        dispatch_x(xdt, [&](auto tag) {
            using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
            k_dx_add<S><<<(unsigned)cdiv(rows * D, 256), 256, 0, st>>>(static_cast<S*>(dx), graw, w,
                                                                       rows, (int)D);
        });
        SKB_CHECK_LAUNCH();
    }
}

}  // namespace skb
