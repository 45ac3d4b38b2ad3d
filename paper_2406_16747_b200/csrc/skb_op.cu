// The SparseK operator on rows of a batch: sparsek / sparsek_jvp / topk_hard
// (proj/src/sparsek_op.cpp:102-165). One CTA per row: descending sort of the
// row in shared memory (global scratch above 8192 entries), exclusive prefix
// sums, the exact breakpoint solve shared with K2 (skb_solve.cuh), then
// finish() — membership decided by value (sparsek_op.cpp:36-57).
#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_solve.cuh"

namespace skb {

namespace {

constexpr int kOpThreads = 256;
constexpr int kSmemCap = 8192;

struct OpArgs {
    const double* z;
    const double* v;
    double* p;
    double* out;
    double* tau;
    int64_t* u_count;
    int64_t* w_count;
    int32_t* flags;
    double* scratch;  // per-row scratch for m > kSmemCap: [n2 + m + 1] per concurrent row
    int m, n2;
    double k;
    int mode;  // 0 sparsek, 1 jvp
};

__global__ void __launch_bounds__(kOpThreads) k_sparsek_rows(OpArgs a) {
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ int cnt[3];
    const int row = blockIdx.x;
    const double* z = a.z + (int64_t)row * a.m;
    double* bz;
    double* P;
    if (a.scratch) {
        bz = a.scratch + (int64_t)row * (a.n2 + a.m + 1);
        P = bz + a.n2;
    } else {
        bz = sm;
        P = sm + a.n2;
    }
    const int m = a.m;
    if ((double)m < a.k) {  // infeasible: all ones, tau = -inf (sparsek_op.cpp:21-32, :108)
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            if (a.mode == 0) a.p[(int64_t)row * m + j] = 1.0;
            else a.out[(int64_t)row * m + j] = 0.0;
        }
        if (threadIdx.x == 0 && a.mode == 0) {
            a.tau[row] = -INFINITY;
            a.u_count[row] = m;
            a.w_count[row] = m;
            a.flags[row] = 3;
        }
        return;
    }
    for (int i = threadIdx.x; i < a.n2; i += blockDim.x) bz[i] = i < m ? z[i] : -INFINITY;
    __syncthreads();
    bitonic_desc(bz, a.n2);
    excl_prefix(bz, P, m, red);
    int frac;
    const double tau = solve_sorted(bz, P, m, a.k, red, &frac);
    if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
    __syncthreads();
    int uc = 0, wc = 0, sc = 0;
    double vs = 0.0;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        double pj = z[j] - tau;
        pj = pj < 0.0 ? 0.0 : (pj > 1.0 ? 1.0 : pj);
        if (a.mode == 0) a.p[(int64_t)row * m + j] = pj;
        if (pj == 1.0) {
            ++uc;
            ++wc;
        } else if (pj > 0.0) {
            ++wc;
            ++sc;
            if (a.mode == 1) vs += a.v[(int64_t)row * m + j];
        }
    }
    atomicAdd(&cnt[0], uc);
    atomicAdd(&cnt[1], wc);
    atomicAdd(&cnt[2], sc);
    double vsum = 0.0;
    if (a.mode == 1) {
        vsum = warp_sum(vs);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = vsum;
        __syncthreads();
        vsum = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) vsum += red[w];
    }
    __syncthreads();
    if (a.mode == 1) {
        const int ns = cnt[2];
        const double vbar = ns ? vsum / (double)ns : 0.0;
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            double pj = z[j] - tau;
            pj = pj < 0.0 ? 0.0 : (pj > 1.0 ? 1.0 : pj);
            a.out[(int64_t)row * m + j] = (ns && pj > 0.0 && pj < 1.0) ? a.v[(int64_t)row * m + j] - vbar : 0.0;
        }
    } else if (threadIdx.x == 0) {
        a.tau[row] = tau;
        a.u_count[row] = cnt[0];
        a.w_count[row] = cnt[1];
        a.flags[row] = cnt[2] == 0 ? 1 : 0;
    }
}

// topk_hard: element i is kept iff fewer than k elements rank ahead of it
// (larger value, or equal value and lower index) — sparsek_op.cpp:152-165.
__global__ void __launch_bounds__(256)
k_topk_rows(const double* __restrict__ z, int m, int64_t k, double* __restrict__ out) {
    __shared__ double tile[1024];
    const int row = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double* zr = z + (int64_t)row * m;
    const double zi = i < m ? zr[i] : 0.0;
    int64_t ahead = 0;
    for (int c0 = 0; c0 < m; c0 += 1024) {
        for (int t = threadIdx.x; t < 1024; t += blockDim.x) tile[t] = c0 + t < m ? zr[c0 + t] : 0.0;
        __syncthreads();
        if (i < m) {
            const int n = min(1024, m - c0);
            for (int t = 0; t < n; ++t) {
                const double x = tile[t];
                ahead += (x > zi) || (x == zi && c0 + t < i);
            }
        }
        __syncthreads();
    }
    if (i < m) out[(int64_t)row * m + i] = (k >= m || ahead < k) ? 1.0 : 0.0;
}

int next_pow2(int x) {
    int n = 1;
    while (n < x) n <<= 1;
    return n;
}

void launch_rows(OpArgs a, int64_t n, cudaStream_t st) {
    a.n2 = next_pow2(std::max(a.m, 1));
    size_t smem = 0;
    double* scratch = nullptr;
    if (a.n2 <= kSmemCap) {
        smem = (size_t)(a.n2 + a.m + 1) * sizeof(double);
        static uint64_t attr = 0;
        if (first_on_device(&attr)) {
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_sparsek_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)((2 * kSmemCap + 1) * sizeof(double))));
        }
    } else {
        SKB_CHECK_CUDA(cudaMallocAsync(&scratch, (size_t)n * (a.n2 + a.m + 1) * sizeof(double), st));
    }
    a.scratch = scratch;
    k_sparsek_rows<<<(unsigned)n, kOpThreads, smem, st>>>(a);
    SKB_CHECK_LAUNCH();
    if (scratch) SKB_CHECK_CUDA(cudaFreeAsync(scratch, st));
}

}  // namespace

void run_sparsek(int64_t n, int64_t m, const double* z, double k, double* p, double* tau,
                 int64_t* uc, int64_t* wc, int32_t* flags, cudaStream_t st) {
    SKB_REQUIRE(m >= 1 && n >= 1, SKB_EARG, "sparsek: empty input");
    SKB_REQUIRE(k > 0.0 && std::isfinite(k), SKB_EARG, "KBudget: k must be positive and finite");
    SKB_REQUIRE(m < (int64_t(1) << 28), SKB_ESHAPE, "sparsek: row too long");
    OpArgs a{};
    a.z = z;
    a.p = p;
    a.tau = tau;
    a.u_count = uc;
    a.w_count = wc;
    a.flags = flags;
    a.m = (int)m;
    a.k = k;
    a.mode = 0;
    launch_rows(a, n, st);
}

void run_sparsek_jvp(int64_t n, int64_t m, const double* z, double k, const double* v, double* out,
                     cudaStream_t st) {
    SKB_REQUIRE(m >= 1 && n >= 1, SKB_EARG, "sparsek: empty input");
    SKB_REQUIRE(k > 0.0 && std::isfinite(k), SKB_EARG, "KBudget: k must be positive and finite");
    OpArgs a{};
    a.z = z;
    a.v = v;
    a.out = out;
    a.m = (int)m;
    a.k = k;
    a.mode = 1;
    launch_rows(a, n, st);
}

// sparsek_jvp(sol, v) (proj/src/sparsek_op.cpp:141-150) from a solution's p:
// out_j = v_j - mean over the support {0 < p < 1} on the support, else 0.
__global__ void __launch_bounds__(1024) k_support_jvp(const double* __restrict__ p, const double* __restrict__ v,
                                                      int m, double* __restrict__ out) {
    __shared__ double ssum[32];
    __shared__ int scnt[32];
    double s = 0.0;
    int c = 0;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const bool sup = p[j] > 0.0 && p[j] < 1.0;
        s += sup ? v[j] : 0.0;
        c += sup;
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) {
        ssum[threadIdx.x >> 5] = s;
        scnt[threadIdx.x >> 5] = c;
    }
    __syncthreads();
    double tot = 0.0;
    int cnt = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {  // fixed order: deterministic
        tot += ssum[w];
        cnt += scnt[w];
    }
    const double vbar = cnt ? tot / (double)cnt : 0.0;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const bool sup = p[j] > 0.0 && p[j] < 1.0;
        out[j] = sup ? v[j] - vbar : 0.0;
    }
}

void run_support_jvp(int64_t m, const double* p, const double* v, double* out, cudaStream_t st) {
    SKB_REQUIRE(m >= 0, SKB_ESHAPE, "sparsek_jvp: v length mismatch");
    if (m == 0) return;
    k_support_jvp<<<1, 1024, 0, st>>>(p, v, (int)m, out);
    SKB_CHECK_LAUNCH();
}

void run_topk_hard(int64_t n, int64_t m, const double* z, int64_t k, double* out, cudaStream_t st) {
    SKB_REQUIRE(m >= 1 && n >= 1, SKB_EARG, "topk_hard: empty input");
    dim3 g((unsigned)cdiv(m, 256), (unsigned)n);
    k_topk_rows<<<g, 256, 0, st>>>(z, (int)m, k, out);
    SKB_CHECK_LAUNCH();
}

}  // namespace skb
