/* sparsek_b200.h — the C-ABI drop-in boundary of the B200 SparseK attention path.
 *
 * Plain pointers and sizes only; every call takes a cudaStream_t (passed as
 * void*) and returns an skb_status. Errors never fall back to a CPU path: a
 * failing call returns non-zero and skb_last_error() (thread-local) says why.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to the reference tree, proj/...):
 *
 *   skb_score_fwd      detail::score_one / score_tokens
 *                      proj/include/sparsek/selection.hpp:55-56,69-96,
 *                      TimestepNormState::push proj/src/selection.cpp:13-20
 *   skb_score_bwd      scores->raw pullback + dw_score + the dx term
 *                      proj/src/attention.cpp:482-516,564
 *   skb_select         StreamState::push (prefix tau) proj/src/stream.cpp:72-152 +
 *                      SparseKvCache::exit_window/admit_to_cache (top-floor(k)
 *                      retention) proj/src/cache.cpp:136-179 + snapshot/gates :285-311
 *   skb_attn_fwd       SparseKvCache::forward_chunk pass 2 proj/src/cache.cpp:315-394
 *                      (the attention inside sparsek_attention, attention.hpp:81-85)
 *   skb_attn_bwd       sparsek_attention_backward core proj/src/attention.cpp:259-316
 *                      + selection pullback (JVP) :447-479
 *   skb_sparsek*       sparsek / sparsek_jvp / topk_hard
 *                      proj/include/sparsek/sparsek_op.hpp:47-66
 *   skb_cache_*        SparseKvCache + generate_step proj/include/sparsek/cache.hpp:21-102,
 *                      proj/src/cache.cpp:570-577
 *
 * Tensor layout: Q/K/V/O/dO/dQ/dK/dV are [B, L, H, p] contiguous — the
 * reference's row-major [L, D] per sequence with head h in columns
 * [h*p, (h+1)*p) (proj/include/sparsek/attention.hpp:36). Scores u are
 * float64 [B, L], as the reference keeps them (selection.hpp:72-74).
 */
#ifndef SPARSEK_B200_H
#define SPARSEK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference error taxonomy (proj/include/sparsek/common.hpp:9-25). */
typedef enum {
    SKB_OK = 0,
    SKB_ESHAPE = 1,    /* ShapeError    */
    SKB_EARG = 2,      /* ArgumentError */
    SKB_ENUMERIC = 3,  /* NumericError  */
    SKB_ECONFIG = 4,   /* ConfigError   */
    SKB_EIO = 5,       /* IoError       */
    SKB_ECUDA = 6      /* CUDA runtime / launch failure */
} skb_status;

typedef enum { SKB_F32 = 0, SKB_BF16 = 1, SKB_F64 = 2 } skb_dtype;

/* Execution-path flags. The tensor-core (tcgen05) path is used for BF16 by
 * default; F32/F64 always run the CUDA-core gather path. */
#define SKB_FLAG_FORCE_GATHER 1u /* run BF16 on the CUDA-core gather kernels */
#define SKB_FLAG_LINEAR_MIX 2u   /* AttnConfig::linear_mix: window = floor(k) = 0 is allowed
                                    (the linear branch reaches every position) */

/* AttnConfig (proj/include/sparsek/attention.hpp:18-32) at the Q/K/V/u level. */
typedef struct skb_attn_desc {
    int64_t batch;     /* B: independent sequences                      */
    int64_t seq_len;   /* L                                             */
    int64_t heads;     /* H                                             */
    int64_t head_dim;  /* p = d_model / heads                           */
    double k;          /* selection budget (real); 0 = pure window      */
    int64_t window;    /* sliding-window size w                         */
    double scale;      /* 0 -> 1/sqrt(p)                                */
    int32_t key_mode;  /* 0 KeyMode::hard, 1 KeyMode::soft              */
    int32_t mask_mode; /* 0 MaskApply::soft, 1 MaskApply::straight_through */
    int32_t dtype;     /* skb_dtype of Q/K/V/O/dO/dQ/dK/dV             */
    uint32_t flags;    /* SKB_FLAG_*                                    */
    int64_t chunk_len; /* 0: one chunk; > 0: chunk-wise recurrent training
                          (chunked_forward, Algorithm 3): the forward is
                          unchanged, gradients never cross to the left of a
                          chunk start (proj/src/attention.cpp:228-234)     */
} skb_attn_desc;

/* ScoringParams (proj/include/sparsek/selection.hpp:19-27) minus w_score. */
typedef struct skb_scoring {
    int32_t norm_mode;     /* 0 none, 1 timestep_norm                   */
    int32_t slope_order;   /* 0 slope_then_norm, 1 norm_then_slope      */
    int32_t slope_enabled; /* 0/1                                       */
    int32_t chunk_len;     /* backward only: the norm pullback stays inside
                              each chunk (proj/src/attention.cpp:482-502); 0 = one chunk */
    double slope_eps;      /* > 0                                       */
} skb_scoring;

/* Where skb_select puts its products inside the caller's workspace (byte
 * offsets). leave[b*L + j] = the push time at which position j leaves the
 * top-floor(k) set (== j when it never enters, == L-w when it never leaves);
 * tau[b*L + t] = the threshold after push t (-inf while t+1 < k); nfrac is the
 * fractional-support size |{j<=t : 0 < u_j - tau_t < 1}|; qb_list holds, per
 * 128-query block, the ascending union of the selected sets its queries read. */
typedef struct skb_select_layout {
    uint64_t leave;       /* int32  [B, L]                 */
    uint64_t leave_ceil;  /* int32  [B, L] (rank ceil(k))  */
    uint64_t tau;         /* double [B, L]  (push time)    */
    uint64_t nfrac;       /* int32  [B, L]  (push time)    */
    uint64_t qb_count;    /* int32  [B, NQB]               */
    uint64_t qb_list;     /* int32  [B, NQB, qb_cap]       */
    uint64_t ever_count;  /* int32  [B]                    */
    uint64_t ever_list;   /* int32  [B, L] ever-selected keys, ascending */
    uint64_t misc;        /* int32 scratch (overflow queue) */
    uint64_t scratch;     /* double scratch (overflow chunks) */
    uint64_t uf;          /* float  [B, L]  u as fp32 (tensor-core gates)    */
    uint64_t tauf;        /* float  [B, L]  tau as fp32 (push time)          */
    uint64_t qb_leave;    /* int32  [B, NQB, qb_cap] leave - key of each union entry (0 = padding) */
    uint64_t qb_uf;       /* float  [B, NQB, qb_cap] u of each union entry     */
    uint64_t qb_flags;    /* int32x4 [B, NQB, qb_cap/128] per 128-entry tile (.x used):
                             bit0 every key valid for every query of the block,
                             bit1 every gate saturated (u >= tau(t_hi) + 1)   */
    uint64_t total_bytes;
    int64_t qblock;       /* queries per block (128)       */
    int64_t nqb;          /* ceil(L / qblock)              */
    int64_t qb_cap;       /* floor(k) + qblock rounded up to a multiple of 128 (list padded with -1) */
} skb_select_layout;

const char* skb_last_error(void);
int skb_version(void);

/* ---- K1: scoring (raw = x.w in float64, Welford prefix norm, slope) ------ */
/* x: [B, L, D] of x_dtype; w: float64 [D]; outputs float64 [B, L]. Exact
 * sequential Welford order per sequence (bit-identical arithmetic to the
 * reference when x rows and w match). */
int skb_score_fwd(int64_t B, int64_t L, int64_t D, int32_t x_dtype, const void* x,
                  const double* w, const skb_scoring* sc, double* raw, double* u, double* mean,
                  double* sdev, void* stream);
/* The scoring GEMV alone: raw[r] = sum_c x[r, c] * w[c] for `rows` rows of
 * x [rows, D] (the raw part of detail::score_one,
 * proj/include/sparsek/selection.hpp:72-74: left to right, float64, no fma).
 * Enqueued on `stream`, no host synchronisation. */
int skb_score_raw(int64_t rows, int64_t D, int32_t x_dtype, const void* x, const double* w, double* raw,
                  void* stream);
/* The fused front of forward_chunk for bf16 (proj/src/cache.cpp:204-228):
 * q|k|v = x Wq|Wk|Wv (x [B*L, D], W* [D, D], outputs [B*L, D]; D a multiple of
 * 256) as one hand-written tcgen05 GEMM that also forms raw = x . w_score
 * (bit-identical to skb_score_raw) from the same x tiles, and the rest of
 * skb_score_fwd (Welford prefix norm + slope) streaming under it. w_score NULL:
 * projections only (scores idle, k = 0). Synchronises `stream`. */
int skb_proj_score(int64_t B, int64_t L, int64_t D, const void* x, const void* wq, const void* wk, const void* wv,
                   const double* w_score, const skb_scoring* sc, void* q, void* k, void* v, double* raw, double* u,
                   double* mean, double* sdev, void* stream);
/* Incremental scoring (score_tokens with base_pos: the TimestepNormState is
 * carried across calls, proj/include/sparsek/selection.hpp:55-56,
 * proj/src/selection.cpp:13-31): x [B, n, D] continues each sequence's
 * float64 state [B, 3] = {count, mean, m2} (zeros for a fresh sequence);
 * raw/u float64 [B, n]. Bit-identical to the reference for identical x and w. */
int skb_score_continue(int64_t B, int64_t n, int64_t D, int32_t x_dtype, const void* x,
                       const double* w, const skb_scoring* sc, double* state, double* raw,
                       double* u, void* stream);
/* gu: float64 [B, L] -> graw [B, L]; dw_score float64 [D] (= sum over B and
 * positions of graw * x); dx (optional, x_dtype [B, L, D]) += graw * w. */
int skb_score_bwd(int64_t B, int64_t L, int64_t D, int32_t x_dtype, const void* x,
                  const double* w, const skb_scoring* sc, const double* gu, const double* raw,
                  const double* mean, const double* sdev, double* graw, double* dw_score,
                  void* dx, void* stream);

/* ---- K2: prefix SparseK threshold + top-floor(k) retention --------------- */
int skb_select_layout_of(const skb_attn_desc* d, skb_select_layout* out);
int skb_select(const skb_attn_desc* d, const double* u, void* ws, void* stream);

/* ---- K3/K4: gated sparse attention over Sel_i U window ------------------- */
/* lse: float64 [B, H, L] = maxa + log(denom) per (query, head). */
int skb_attn_fwd(const skb_attn_desc* d, const void* q, const void* k, const void* v,
                 const double* u, const void* sel_ws, void* o, double* lse, void* stream);
int skb_attn_bwd_workspace_size(const skb_attn_desc* d, size_t* bytes);
/* du: float64 [B, L] gradient w.r.t. the scores u (selection JVP included). */
int skb_attn_bwd(const skb_attn_desc* d, const void* q, const void* k, const void* v,
                 const void* o, const void* dout, const double* lse, const double* u,
                 const void* sel_ws, void* dq, void* dk, void* dv, double* du, void* ws,
                 void* stream);

/* ---- Linear-attention mix (Appendix B.1) --------------------------------- */
/* linear_mix_attention (proj/include/sparsek/attention.hpp:93-99): exact
 * attention over the SparseK snapshot (selected keys with gate m = g, window
 * m = 1) mixed with positive-feature linear attention over every causal
 * position, phi(z) = elu(F_h z) + 1:
 *   o_i = sum_{j<=i} w_ij v_j / sum_{j<=i} w_ij,
 *   w_ij = (1 - m_ij) phi(q_i).phi(k_j) + m_ij exp(scale q_i.k_j)
 * (forward proj/src/cache.cpp:262-278,322-356; backward
 * proj/src/attention.cpp:317-445,519-549). dtype float32 or float64 (the
 * reference's instantiations); feat / dfeat: float64 [H, p, p]; den: float64
 * [B, H, L] (saved by the forward for the backward); ws: the workspace of
 * skb_linmix_workspace_size (both calls). A nonpositive denominator is
 * SKB_ENUMERIC, as the reference's NumericError. */
int skb_linmix_workspace_size(const skb_attn_desc* d, size_t* bytes);
int skb_linmix_fwd(const skb_attn_desc* d, const void* q, const void* k, const void* v, const double* u,
                   const void* sel_ws, const double* feat, void* o, double* den, void* ws, void* stream);
int skb_linmix_bwd(const skb_attn_desc* d, const void* q, const void* k, const void* v, const double* u,
                   const void* sel_ws, const double* feat, const double* den, const void* dout, void* dq,
                   void* dk, void* dv, double* du, double* dfeat, void* ws, void* stream);

/* phi(z) = elu(F_h z) + 1 per row of z [rows, H, p] (float32/float64), feat
 * float64 [H, p, p] -> out float64 [rows, H, p]. */
int skb_linmix_phi(int64_t rows, int64_t heads, int64_t head_dim, int32_t dtype, const void* z, const double* feat,
                   double* out, void* stream);

/* ---- SparseK operator (batched rows) ------------------------------------ */
/* z: float64 [n, m]; p: [n, m]; tau: [n] (-inf when infeasible); counts [n];
 * flags[n]: bit0 degenerate, bit1 infeasible. */
int skb_sparsek(int64_t n, int64_t m, const double* z, double k, double* p, double* tau,
                int64_t* u_count, int64_t* w_count, int32_t* flags, void* stream);
int skb_sparsek_jvp(int64_t n, int64_t m, const double* z, double k, const double* v,
                    double* out, void* stream);
int skb_topk_hard(int64_t n, int64_t m, const double* z, int64_t k, double* out, void* stream);
/* sparsek_jvp(sol, v) from a solution's weights p (proj/src/sparsek_op.cpp:141-150):
 * out = (v - mean over {0 < p < 1} of v) on that support, 0 elsewhere; device [m]. */
int skb_support_jvp(int64_t m, const double* p, const double* v, double* out, void* stream);
/* Row-major C[M, N] = A[M, K] B[K, N] on the device (the reference's matmul,
 * proj/src/numerics.cpp:8-24; a library GEMM), dtype F32/F64/BF16. */
int skb_matmul(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* a, const void* b, void* c, void* stream);

/* ---- K5: constant-(floor(k)+w) KV cache for decoding --------------------- */
typedef struct skb_cache skb_cache;
/* d->seq_len = maximum number of positions a sequence may see. */
int skb_cache_create(const skb_attn_desc* d, skb_cache** out);
int skb_cache_destroy(skb_cache* c);
/* One decode step for all B sequences: q/k/v [B, H, p] (dtype), u float64 [B]
 * (the new tokens' frozen scores) -> o [B, H, p]. */
int skb_cache_step(skb_cache* c, const void* q, const void* k, const void* v, const double* u,
                   void* o, void* stream);
/* Linear-attention mix decode (a cache created with SKB_FLAG_LINEAR_MIX,
 * float32/float64; SparseKvCache::forward_chunk with LinearMixParams,
 * proj/src/cache.cpp:262-278,322-356): skb_cache_linmix_prefill after
 * skb_cache_prefill(k, v, u, n) records phi(k) of the retained rows and adds
 * the n positions to the prefix state M = sum phi(k) v^T, b = sum phi(k);
 * skb_cache_linmix_step = one position (stream push, eviction, state update)
 * and the mixture readout o [B, H, p]. phq/phk: float64 phi rows
 * (skb_linmix_phi). A nonpositive denominator is SKB_ENUMERIC. */
int skb_cache_linmix_prefill(skb_cache* cache, const void* v, const double* phk, int64_t n, void* stream);
int skb_cache_linmix_step(skb_cache* cache, const void* q, const void* k, const void* v, const double* u,
                          const double* phq, const double* phk, void* o, void* stream);
/* Append n positions per sequence without attending (a prompt prefill):
 * k/v [B, n, H, p] (dtype), u float64 [B, n]. The selection state advances
 * exactly as n decode steps would (forward_chunk pass 1,
 * proj/src/cache.cpp:259-311); only the rows still retained afterwards are
 * copied into the slot pool. */
int skb_cache_prefill(skb_cache* c, const void* k, const void* v, const double* u, int64_t n,
                      void* stream);
/* Host-visible state for tests/inspection: retained positions (ascending
 * selected then window), count, tau, positions seen, peak retained. */
/* SparseKvCache<T>::serialize / deserialize (proj/src/cache.cpp:416-545) of
 * sequence b: the reference's snapshot payload (without the "SPKC" file header
 * of save_cache_snapshot, :579-618). norm_state = the TimestepNormState
 * {count, mean, m2} of the caller's scoring (the cache works at the q/k/v/u
 * level; null on snapshot = a fresh state). Snapshot with out == NULL returns
 * the size in *bytes. Restore overwrites sequence b of a cache of the same
 * configuration and returns the norm state. */
int skb_cache_snapshot(skb_cache* c, int64_t b, const double* norm_state, uint8_t* out, size_t* bytes,
                       void* stream);
int skb_cache_restore(skb_cache* c, int64_t b, const uint8_t* data, size_t bytes, double* norm_state,
                      void* stream);
int skb_cache_state(skb_cache* c, int64_t b, int32_t* positions, int64_t* count, double* tau,
                    int64_t* seen, int64_t* peak, void* stream);
/* The eviction ledger of sequence b (SparseKvCache::drain_evictions / ever_evicted /
 * frozen_score, proj/include/sparsek/cache.hpp:38-48): pending evictions since the
 * last drain (cleared when drain != 0; *n_pending = their count, the first
 * pending_cap are copied), the evicted flag of positions [0, evicted_cap) and
 * the frozen scores of positions [0, scores_cap). Host outputs; any may be NULL. */
int skb_cache_ledger(skb_cache* c, int64_t b, int32_t drain, int64_t* pending, int64_t pending_cap,
                     int64_t* n_pending, uint8_t* evicted, int64_t evicted_cap, double* scores, int64_t scores_cap,
                     void* stream);


/* ---- Incremental SparseK stream on the device (Algorithm 2) ------------- */
/* StreamState (proj/include/sparsek/stream.hpp:26-72, proj/src/stream.cpp:72-192):
 * the same push/scan, with the survivors kept as a sorted device array. */
typedef struct skb_stream skb_stream;
typedef struct skb_stream_info {
    double tau;          /* -inf while t < k                         */
    int64_t t;           /* elements pushed                           */
    int64_t survivors;   /* |heap_s|                                  */
    int64_t saturated;   /* |heap_f|                                  */
    uint64_t cap_drops;  /* survivors dropped by a bounded heap       */
    uint64_t heap_ops;
    double k;
} skb_stream_info;
/* capacity = maximum number of pushes; heap_cap 0 = unbounded. */
int skb_stream_create(double k, int64_t heap_cap, int64_t capacity, skb_stream** out);
int skb_stream_destroy(skb_stream* s);
/* Push z[0..n) (device float64) in order; per push the threshold after it and
 * whether it entered the survivors (device outputs, either may be NULL). */
int skb_stream_push(skb_stream* s, const double* z, int64_t n, double* tau_out,
                    uint8_t* inserted_out, void* stream);
int skb_stream_query(skb_stream* s, skb_stream_info* out, void* stream);
/* StreamState::push(z) with its StreamStepResult (proj/include/sparsek/stream.hpp:12-18,
 * proj/src/stream.cpp:72-152) in one device round trip: z is a host value;
 * evicted (host, max_evicted entries) receives the indices that left the
 * survivors during this push, in pop order; n_evicted is their total count. */
typedef struct skb_stream_step {
    double tau;         /* -inf while t < k                            */
    int64_t t;          /* elements pushed so far                       */
    int32_t inserted;   /* 0: arrived at or below tau, never survived   */
    int32_t cap_forced; /* a bounded heap dropped a survivor            */
    int64_t n_evicted;
} skb_stream_step;
int skb_stream_push_step(skb_stream* s, double z, skb_stream_step* out, int64_t* evicted, int64_t max_evicted,
                         void* stream);
/* StreamState::solution + stream_mask (proj/src/stream.cpp:154-222) on the
 * device: survivors in ascending index order — p (float64), indices (int64)
 * and, when hard != NULL, the top-floor(k) SelectionMask flag (uint8); all
 * device buffers with room for every survivor. Counts and tau on the host. */
typedef struct skb_stream_solution_info {
    double tau;          /* -inf when infeasible (t < k)                */
    int64_t t, n;        /* pushes; survivors (entries written)        */
    int64_t u_count, w_count;
    int32_t degenerate, infeasible;
} skb_stream_solution_info;
int skb_stream_solution(skb_stream* s, double* p, int64_t* indices, uint8_t* hard, skb_stream_solution_info* out,
                        void* stream);
/* Host copies: survivor values/indices in ascending index order (|survivors|
 * entries) and the evicted flag of every pushed index (t entries). */
/* The reference's stream wire format (StreamState::serialize/deserialize,
 * proj/src/stream.cpp:224-289; little-endian k, heap_cap, tau, t, sum_s,
 * sum_f, cap_drops, heap_ops, pushes_since_refresh, heap S, heap F, evicted
 * bits). serialize: out == NULL returns the size in *bytes; the heaps are
 * written in (value asc, index desc) order, a valid heap for the reference's
 * HeapCmp. deserialize: a blob of either origin -> a new device stream with
 * room for `capacity` pushes in total. */
int skb_stream_serialize(skb_stream* s, uint8_t* out, size_t* bytes, void* stream);
int skb_stream_deserialize(const uint8_t* data, size_t bytes, int64_t capacity, skb_stream** out);
int skb_stream_survivors(skb_stream* s, double* values, int64_t* indices, uint8_t* evicted,
                         void* stream);

/* ---- x-level operator: sparsek_attention<T> / sparsek_attention_backward<T>
 * (proj/include/sparsek/attention.hpp:81-91, proj/src/attention.cpp:37-43,214-575)
 * and SparseKvCache<T>::forward_chunk / generate_step (proj/include/sparsek/
 * cache.hpp:21-102). x [B, L, d_model] and W* [d_model, d_model] (row-major,
 * head h owns columns [h*p, (h+1)*p)) in `dtype`; w_score float64 [d_model].
 * All pointers are device (or managed) memory; projections are library GEMMs. */
typedef struct skb_x_desc {
    int64_t batch;      /* B independent sequences                         */
    int64_t seq_len;    /* L (for a cache: the maximum positions per sequence) */
    int64_t d_model;    /* D = heads * head_dim                            */
    int64_t heads;
    double k;           /* AttnConfig::k                                   */
    int64_t window;     /* AttnConfig::window                              */
    double scale;       /* 0 -> 1/sqrt(head_dim)                           */
    int32_t key_mode;   /* 0 hard, 1 soft                                  */
    int32_t mask_mode;  /* 0 soft, 1 straight_through                      */
    int32_t dtype;      /* skb_dtype of x, W*, y and the gradients         */
    uint32_t flags;     /* SKB_FLAG_*                                      */
    int64_t chunk_len;  /* chunked_forward's stop-grad chunks; 0 = one     */
    skb_scoring scoring;
} skb_x_desc;

typedef struct skb_xattn skb_xattn; /* a device-resident AttnTape */
/* y = sparsek_attention(x); with tape != NULL the forward state is kept in a
 * new tape (free with skb_xattn_destroy). */
int skb_xattn_forward(const skb_x_desc* d, const void* x, const void* wq, const void* wk, const void* wv,
                      const void* wo, const double* w_score, void* y, skb_xattn** tape, void* stream);
/* AttnGrads from a tape: dx [B, L, D], dW* [D, D] (dtype), dw_score float64 [D]. */
int skb_xattn_backward(skb_xattn* tape, const void* grad_out, const void* wq, const void* wk, const void* wv,
                       const void* wo, const double* w_score, void* dx, void* dwq, void* dwk, void* dwv,
                       void* dwo, double* dw_score, void* stream);
/* linear_mix_attention (proj/include/sparsek/attention.hpp:93-99) and its
 * backward with LinearMixParams: d->flags carries SKB_FLAG_LINEAR_MIX (the
 * scoring must be timestep_norm), feat / dfeat float64 [H, p, p]. The tape's
 * lse field then holds the mixture denominators. */
int skb_xattn_forward_lin(const skb_x_desc* d, const void* x, const void* wq, const void* wk, const void* wv,
                          const void* wo, const double* w_score, const double* feat, void* y, skb_xattn** tape,
                          void* stream);
int skb_xattn_backward_lin(skb_xattn* tape, const void* grad_out, const void* wq, const void* wk, const void* wv,
                           const void* wo, const double* w_score, const double* feat, void* dx, void* dwq,
                           void* dwk, void* dwv, void* dwo, double* dw_score, double* dfeat, void* stream);
/* Copy one AttnTape field (host or device destination, `bytes` = its size):
 * x/q/k/v/head_concat [B, L, D] dtype; raw/u/norm_mean/norm_sdev float64 [B, L];
 * lse float64 [B, H, L] (= maxa + log denom); tau_push float64 [B, L] (push
 * time t; -inf while t + 1 < k); leave int32 [B, L] (position j is selected for
 * push times j <= t < leave_j). */
enum {
    SKB_TAPE_X = 0, SKB_TAPE_Q, SKB_TAPE_K, SKB_TAPE_V, SKB_TAPE_HEAD_CONCAT, SKB_TAPE_RAW, SKB_TAPE_U,
    SKB_TAPE_NORM_MEAN, SKB_TAPE_NORM_SDEV, SKB_TAPE_LSE, SKB_TAPE_TAU_PUSH, SKB_TAPE_LEAVE
};
int skb_xattn_tape_get(skb_xattn* tape, int32_t field, void* dst, size_t bytes, void* stream);
int skb_xattn_destroy(skb_xattn* tape);

typedef struct skb_xcache skb_xcache; /* SparseKvCache<T> for B sequences */
int skb_xcache_create(const skb_x_desc* d, skb_xcache** out);
int skb_xcache_destroy(skb_xcache* c);
/* forward_chunk: x [B, n, D] -> y [B, n, D]; generate_step is n = 1. */
int skb_xcache_forward_chunk(skb_xcache* c, const void* x, int64_t n, const void* wq, const void* wk,
                             const void* wv, const void* wo, const double* w_score, void* y, void* stream);
/* The same with LinearMixParams (a cache created with SKB_FLAG_LINEAR_MIX;
 * feat float64 [H, p, p]). */
int skb_xcache_forward_chunk_lin(skb_xcache* c, const void* x, int64_t n, const void* wq, const void* wk,
                                 const void* wv, const void* wo, const double* w_score, const double* feat, void* y,
                                 void* stream);
/* The underlying q/k/v-level cache (skb_cache_state / snapshot / restore). */
skb_cache* skb_xcache_inner(skb_xcache* c);
/* TimestepNormState {count, mean, m2} per sequence (host [B, 3]): get (set = 0) or set. */
int skb_xcache_norm_state(skb_xcache* c, double* norm_state, int32_t set, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEK_B200_H */
