// The extern "C" boundary (include/sparsek_b200.h): argument checks, error
// mapping onto the reference's taxonomy, and dispatch to the kernels.
#include <cstdio>
#include <string>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {
void run_score_raw(int64_t rows, int64_t D, int32_t xdt, const void* x, const double* w, double* raw,
                   cudaStream_t st);
void run_score_fwd(int64_t B, int64_t L, int64_t D, int32_t xdt, const void* x, const double* w,
                   const skb_scoring& sc, double* raw, double* u, double* mean, double* sdev,
                   cudaStream_t st);
void run_score_continue(int64_t B, int64_t n, int64_t D, int32_t xdt, const void* x, const double* w,
                        const skb_scoring& sc, double* state, double* raw, double* u, cudaStream_t st);
void run_score_bwd(int64_t B, int64_t L, int64_t D, int32_t xdt, const void* x, const double* w,
                   const skb_scoring& sc, const double* gu, const double* raw, const double* mean,
                   const double* sdev, double* graw, double* dw, void* dx, cudaStream_t st);
void run_sparsek(int64_t n, int64_t m, const double* z, double k, double* p, double* tau,
                 int64_t* uc, int64_t* wc, int32_t* flags, cudaStream_t st);
void run_sparsek_jvp(int64_t n, int64_t m, const double* z, double k, const double* v, double* out,
                     cudaStream_t st);
void run_topk_hard(int64_t n, int64_t m, const double* z, int64_t k, double* out, cudaStream_t st);
void run_support_jvp(int64_t m, const double* p, const double* v, double* out, cudaStream_t st);
}  // namespace skb

namespace {
thread_local std::string g_err;

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}
}  // namespace

namespace skb {
void set_last_error(const char* msg) { g_err = msg; }
}  // namespace skb

#define SKB_API_BEGIN try {
#define SKB_API_END                                              \
    }                                                            \
    catch (const skb::Error& e) { return fail(e.code, e.what()); } \
    catch (const std::exception& e) { return fail(SKB_ECUDA, e.what()); } \
    return SKB_OK;

#define NONNULL(p, what) SKB_REQUIRE((p) != nullptr, SKB_EARG, what ": null pointer")

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

const char* skb_last_error(void) { return g_err.c_str(); }
int skb_version(void) { return 1; }

int skb_score_fwd(int64_t B, int64_t L, int64_t D, int32_t x_dtype, const void* x, const double* w,
                  const skb_scoring* sc, double* raw, double* u, double* mean, double* sdev,
                  void* stream) {
    SKB_API_BEGIN
    NONNULL(x, "score_fwd x");
    NONNULL(w, "score_fwd w");
    NONNULL(sc, "score_fwd scoring");
    NONNULL(raw, "score_fwd raw");
    NONNULL(u, "score_fwd u");
    NONNULL(mean, "score_fwd mean");
    NONNULL(sdev, "score_fwd sdev");
    skb::run_score_fwd(B, L, D, x_dtype, x, w, *sc, raw, u, mean, sdev, S(stream));
    SKB_API_END
}

int skb_score_raw(int64_t rows, int64_t D, int32_t x_dtype, const void* x, const double* w, double* raw,
                  void* stream) {
    SKB_API_BEGIN
    NONNULL(x, "score_raw x");
    NONNULL(w, "score_raw w");
    NONNULL(raw, "score_raw raw");
    skb::run_score_raw(rows, D, x_dtype, x, w, raw, S(stream));
    SKB_API_END
}

int skb_score_continue(int64_t B, int64_t n, int64_t D, int32_t x_dtype, const void* x, const double* w,
                       const skb_scoring* sc, double* state, double* raw, double* u, void* stream) {
    SKB_API_BEGIN
    NONNULL(x, "score_continue x");
    NONNULL(w, "score_continue w");
    NONNULL(sc, "score_continue scoring");
    NONNULL(state, "score_continue state");
    NONNULL(raw, "score_continue raw");
    NONNULL(u, "score_continue u");
    skb::run_score_continue(B, n, D, x_dtype, x, w, *sc, state, raw, u, S(stream));
    SKB_API_END
}

int skb_score_bwd(int64_t B, int64_t L, int64_t D, int32_t x_dtype, const void* x, const double* w,
                  const skb_scoring* sc, const double* gu, const double* raw, const double* mean,
                  const double* sdev, double* graw, double* dw_score, void* dx, void* stream) {
    SKB_API_BEGIN
    NONNULL(sc, "score_bwd scoring");
    NONNULL(gu, "score_bwd gu");
    NONNULL(graw, "score_bwd graw");
    SKB_REQUIRE(!dw_score || x, SKB_EARG, "score_bwd: dw_score needs x");
    SKB_REQUIRE(!dx || w, SKB_EARG, "score_bwd: dx needs w");
    skb::run_score_bwd(B, L, D, x_dtype, x, w, *sc, gu, raw, mean, sdev, graw, dw_score, dx,
                       S(stream));
    SKB_API_END
}

int skb_select_layout_of(const skb_attn_desc* d, skb_select_layout* out) {
    SKB_API_BEGIN
    NONNULL(d, "select_layout desc");
    NONNULL(out, "select_layout out");
    skb::validate_desc(*d);
    skb::select_layout(*d, *out);
    SKB_API_END
}

int skb_select(const skb_attn_desc* d, const double* u, void* ws, void* stream) {
    SKB_API_BEGIN
    NONNULL(d, "select desc");
    NONNULL(u, "select u");
    NONNULL(ws, "select workspace");
    skb::run_select(*d, u, ws, S(stream));
    SKB_API_END
}

int skb_attn_fwd(const skb_attn_desc* d, const void* q, const void* k, const void* v,
                 const double* u, const void* sel_ws, void* o, double* lse, void* stream) {
    SKB_API_BEGIN
    NONNULL(d, "attn_fwd desc");
    NONNULL(q, "attn_fwd q");
    NONNULL(k, "attn_fwd k");
    NONNULL(v, "attn_fwd v");
    NONNULL(u, "attn_fwd u");
    NONNULL(sel_ws, "attn_fwd select workspace");
    NONNULL(o, "attn_fwd o");
    NONNULL(lse, "attn_fwd lse");
    skb::validate_desc(*d);
    const skb::SelView s = skb::sel_view(*d, sel_ws);
    if (d->dtype == SKB_BF16 && !(d->flags & SKB_FLAG_FORCE_GATHER) && skb::tc_supported(*d))
        skb::run_attn_fwd_tc(*d, q, k, v, u, s, o, lse, nullptr, S(stream));
    else
        skb::run_attn_fwd_gather(*d, q, k, v, u, s, o, lse, S(stream));
    SKB_API_END
}

int skb_attn_bwd_workspace_size(const skb_attn_desc* d, size_t* bytes) {
    SKB_API_BEGIN
    NONNULL(d, "attn_bwd desc");
    NONNULL(bytes, "attn_bwd bytes");
    skb::validate_desc(*d);
    skb::BwdLayout bl;
    skb::bwd_layout(*d, bl);
    *bytes = bl.total;
    SKB_API_END
}

int skb_attn_bwd(const skb_attn_desc* d, const void* q, const void* k, const void* v,
                 const void* o, const void* dout, const double* lse, const double* u,
                 const void* sel_ws, void* dq, void* dk, void* dv, double* du, void* ws,
                 void* stream) {
    SKB_API_BEGIN
    NONNULL(d, "attn_bwd desc");
    NONNULL(q, "attn_bwd q");
    NONNULL(k, "attn_bwd k");
    NONNULL(v, "attn_bwd v");
    NONNULL(dout, "attn_bwd dout");
    NONNULL(lse, "attn_bwd lse");
    NONNULL(u, "attn_bwd u");
    NONNULL(sel_ws, "attn_bwd select workspace");
    NONNULL(dq, "attn_bwd dq");
    NONNULL(dk, "attn_bwd dk");
    NONNULL(dv, "attn_bwd dv");
    NONNULL(du, "attn_bwd du");
    NONNULL(ws, "attn_bwd workspace");
    skb::validate_desc(*d);
    const skb::SelView s = skb::sel_view(*d, sel_ws);
    skb::BwdLayout bl;
    skb::bwd_layout(*d, bl);
    char* base = static_cast<char*>(ws);
    double* rowsum = reinterpret_cast<double*>(base + bl.rowsum);
    double* colsum = reinterpret_cast<double*>(base + bl.colsum);
    double* mp = reinterpret_cast<double*>(base + bl.mean_prefix);
    const size_t BL = (size_t)d->batch * d->seq_len;
    cudaStream_t st = S(stream);
    SKB_CHECK_CUDA(cudaMemsetAsync(rowsum, 0, BL * sizeof(double), st));
    SKB_CHECK_CUDA(cudaMemsetAsync(colsum, 0, BL * sizeof(double), st));
    if (d->dtype == SKB_BF16 && !(d->flags & SKB_FLAG_FORCE_GATHER) && skb::tc_supported(*d)) {
        NONNULL(o, "attn_bwd o");
        skb::run_attn_bwd_tc(*d, q, k, v, o, dout, lse, u, s, dq, dk, dv, rowsum, colsum, ws, bl, st);
    } else {
        skb::run_attn_bwd_gather(*d, q, k, v, dout, lse, u, s, dq, dk, dv, rowsum, colsum, ws, bl, st);
    }
    skb::run_jvp(*d, u, s, rowsum, colsum, mp, reinterpret_cast<double*>(base + bl.chunk_sums), du, st);
    SKB_API_END
}

int skb_sparsek(int64_t n, int64_t m, const double* z, double k, double* p, double* tau,
                int64_t* u_count, int64_t* w_count, int32_t* flags, void* stream) {
    SKB_API_BEGIN
    NONNULL(z, "sparsek z");
    NONNULL(p, "sparsek p");
    NONNULL(tau, "sparsek tau");
    NONNULL(u_count, "sparsek u_count");
    NONNULL(w_count, "sparsek w_count");
    NONNULL(flags, "sparsek flags");
    skb::run_sparsek(n, m, z, k, p, tau, u_count, w_count, flags, S(stream));
    SKB_API_END
}

int skb_sparsek_jvp(int64_t n, int64_t m, const double* z, double k, const double* v, double* out,
                    void* stream) {
    SKB_API_BEGIN
    NONNULL(z, "sparsek_jvp z");
    NONNULL(v, "sparsek_jvp v");
    NONNULL(out, "sparsek_jvp out");
    skb::run_sparsek_jvp(n, m, z, k, v, out, S(stream));
    SKB_API_END
}

int skb_support_jvp(int64_t m, const double* p, const double* v, double* out, void* stream) {
    SKB_API_BEGIN
    NONNULL(p, "sparsek_jvp p");
    NONNULL(v, "sparsek_jvp v");
    NONNULL(out, "sparsek_jvp out");
    skb::run_support_jvp(m, p, v, out, S(stream));
    SKB_API_END
}

int skb_topk_hard(int64_t n, int64_t m, const double* z, int64_t k, double* out, void* stream) {
    SKB_API_BEGIN
    NONNULL(z, "topk_hard z");
    NONNULL(out, "topk_hard out");
    SKB_REQUIRE(k >= 0, SKB_EARG, "topk_hard: k must be >= 0");
    skb::run_topk_hard(n, m, z, k, out, S(stream));
    SKB_API_END
}

}  // extern "C"
