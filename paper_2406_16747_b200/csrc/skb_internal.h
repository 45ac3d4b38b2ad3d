// Internal interfaces shared by the CUDA translation units (not part of the C ABI).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <cmath>

#include "sparsek_b200.h"

namespace skb {

// CTAs of a persistent grid over `items` work items: one per SM; the
// SKB_MAX_CTAS environment variable caps it (tests and the sanitizer use it
// to put many items, and ring wrap-arounds, on every CTA).
int num_sms();
inline int persist_grid(int64_t items) {
    static const int cap = getenv("SKB_MAX_CTAS") ? atoi(getenv("SKB_MAX_CTAS")) : 0;
    int64_t g = items < num_sms() ? items : num_sms();
    if (cap > 0 && g > cap) g = cap;
    return (int)(g > 0 ? g : 1);
}

// SM count of the current device (persistent grids)
inline int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev);
    return cached[dev] > 0 ? cached[dev] : 148;
}
// Function attributes (dynamic shared memory above 48 KB) are per device
// context: true the first time a call site runs on the current device.
inline bool first_on_device(uint64_t* seen) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (*seen & bit) return false;
    *seen |= bit;
    return true;
}
void validate_desc(const skb_attn_desc& d);
void select_layout(const skb_attn_desc& d, skb_select_layout& o);
void run_select(const skb_attn_desc& d, const double* u, void* ws, cudaStream_t st);

// Views into a select workspace.
struct SelView {
    const int* leave;
    const double* tau;  // push-time indexed, monotone after run_select
    const int* nfrac;
    const int* qb_count;
    const int* qb_list;
    const int* ever_count;
    const int* ever_list;
    const float* uf;    // u as fp32 [B, L]
    const float* tauf;  // tau as fp32 [B, L] (push time)
    const int* qb_leave;    // [B, NQB, qb_cap] leave - key of each union entry (0 = padding)
    const float* qb_uf;     // [B, NQB, qb_cap] u of each union entry
    const int* qb_flags;    // [B, NQB, qb_cap / 128] x 4 ints (16-byte records, .x = flags)
    int nqb, qb_cap;
};
SelView sel_view(const skb_attn_desc& d, const void* ws);

struct BwdLayout {
    uint64_t rowsum, colsum, mean_prefix, chunk_sums, dk_acc, dv_acc, dq_acc, sel_items, sel_order, dq32, uni_hi, total;
};
void bwd_layout(const skb_attn_desc& d, BwdLayout& o);

void run_attn_fwd_gather(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                         const double* u, const SelView& s, void* o, double* lse, cudaStream_t st);
void run_attn_bwd_gather(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                         const void* dout, const double* lse, const double* u, const SelView& s,
                         void* dq, void* dk, void* dv, double* rowsum, double* colsum, void* ws,
                         const BwdLayout& bl, cudaStream_t st);
// Tensor-core (tcgen05) path, BF16 only. Returns false when the shape is not supported.
bool tc_supported(const skb_attn_desc& d);
void run_attn_fwd_tc(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                     const double* u, const SelView& s, void* o, double* lse, void* ws,
                     cudaStream_t st);
void run_attn_bwd_tc(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                     const void* o, const void* dout, const double* lse, const double* u,
                     const SelView& s, void* dq, void* dk, void* dv, double* rowsum,
                     double* colsum, void* ws, const BwdLayout& bl, cudaStream_t st);
// du from the gate-gradient row/column sums (selection pullback).
void run_jvp(const skb_attn_desc& d, const double* u, const SelView& s, const double* rowsum,
             const double* colsum, double* mean_prefix, double* chunk_sums, double* du, cudaStream_t st);

}  // namespace skb
