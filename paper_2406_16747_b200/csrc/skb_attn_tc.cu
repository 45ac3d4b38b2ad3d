// K3/K4 tensor-core path (tcgen05 + TMEM) — BF16 only. See DESIGN.md.
#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

bool tc_supported(const skb_attn_desc& d) {
    (void)d;
    return false;  // enabled once the tcgen05 kernels land
}

void run_attn_fwd_tc(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                     const double* u, const SelView& s, void* o, double* lse, void* ws,
                     cudaStream_t st) {
    (void)d; (void)q; (void)k; (void)v; (void)u; (void)s; (void)o; (void)lse; (void)ws; (void)st;
    throw Error(SKB_ECONFIG, "tensor-core path unavailable for this shape");
}

void run_attn_bwd_tc(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                     const void* o, const void* dout, const double* lse, const double* u,
                     const SelView& s, void* dq, void* dk, void* dv, double* rowsum,
                     double* colsum, void* ws, const BwdLayout& bl, cudaStream_t st) {
    (void)d; (void)q; (void)k; (void)v; (void)o; (void)dout; (void)lse; (void)u; (void)s;
    (void)dq; (void)dk; (void)dv; (void)rowsum; (void)colsum; (void)ws; (void)bl; (void)st;
    throw Error(SKB_ECONFIG, "tensor-core path unavailable for this shape");
}

}  // namespace skb
