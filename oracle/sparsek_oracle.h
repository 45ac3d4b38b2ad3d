/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the B200 path.
 *
 * A plain-C restatement of the reference algorithm at the Q/K/V/u ("core")
 * level, each function citing the reference file:line it follows (paths
 * relative to /root/reference/). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it. Parity of this restatement is
 * pinned against the compiled reference (oracle/_ref) and the reference's own
 * known-answer vectors in tests/test_oracle.py.
 *
 * Layout: Q/K/V/O are [L, H, p] row-major (= the reference's [L, D] with head
 * h owning columns [h*p, (h+1)*p), proj/include/sparsek/attention.hpp:36).
 */
#ifndef SPARSEK_ORACLE_H
#define SPARSEK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double k;        /* selection budget (real, >= 0)            */
    int64_t window;  /* sliding window w                          */
    int64_t heads;   /* H                                         */
    double scale;    /* 0 -> 1/sqrt(p)                            */
    int32_t key_soft;  /* KeyMode::soft (logits gated)           */
    int32_t mask_st;   /* MaskApply::straight_through            */
} orc_cfg;

/* Scoring (proj/include/sparsek/selection.hpp:69-96, proj/src/selection.cpp:13-20).
 * norm_mode: 0 none, 1 timestep_norm; slope_order: 0 slope_then_norm, 1 norm_then_slope. */
int orc_score_fwd(const double* x, const double* w, int64_t L, int64_t D, int32_t norm_mode,
                  int32_t slope_order, int32_t slope_enabled, double slope_eps, double* raw,
                  double* u, double* mean, double* sdev);
/* Scores -> raw pullback (proj/src/attention.cpp:482-502), O(L^2) as in the reference. */
void orc_score_bwd(const double* gu, const double* raw, const double* mean, const double* sdev,
                   int64_t L, int32_t norm_mode, double* graw);

/* Batch SparseK (proj/src/sparsek_op.cpp:63-114). Returns 0 or an error code. */
int orc_sparsek(const double* z, int64_t m, double k, double* p, double* tau, int64_t* u_count,
                int64_t* w_count, int32_t* degenerate, int32_t* infeasible);
/* JVP (proj/src/sparsek_op.cpp:141-150). */
int orc_sparsek_jvp(const double* z, int64_t m, double k, const double* v, double* out);
/* Hard top-k, ties to the lower index (proj/src/sparsek_op.cpp:152-165). */
void orc_topk_hard(const double* z, int64_t m, int64_t k, double* out);
/* Incremental stream (proj/src/stream.cpp:72-152): tau after each push. */
int orc_stream_taus(const double* z, int64_t n, double k, double* tau_out, uint8_t* inserted);

/* Retention + snapshot (proj/src/cache.cpp:136-179, 259-311). Per query i:
 * tau_q[i] = stream tau after push i-w (or -inf), n_sel[i] selected entries
 * first (ascending positions), then the window ring (ascending), then self
 * when w == 0 and not selected. gate[] is aligned with att[] (1.0 for
 * non-selected entries). With att == NULL only att_off is filled (sizes). */
int orc_select(const double* u, int64_t L, double k, int64_t window, double* tau_q,
               int32_t* n_sel, int64_t* att_off, int32_t* att, double* gate);

/* Attention forward on the snapshots (proj/src/cache.cpp:358-393). */
int orc_attn_fwd(const double* q, const double* k, const double* v, int64_t L, int64_t p,
                 const orc_cfg* cfg, const int32_t* n_sel, const int64_t* att_off,
                 const int32_t* att, const double* gate, double* o, double* maxa, double* denom);

/* Attention backward (proj/src/attention.cpp:259-316) + selection pullback
 * (proj/src/attention.cpp:447-479). Outputs dq/dk/dv [L,H,p], gu [L] (scores),
 * and gm_rowsum [L] = sum over heads and selected fractional entries of gm
 * (diagnostic). Single chunk (chunk start 0). */
int orc_attn_bwd(const double* q, const double* k, const double* v, const double* dout,
                 int64_t L, int64_t p, const orc_cfg* cfg, const double* u, const double* tau_q,
                 const int32_t* n_sel, const int64_t* att_off, const int32_t* att,
                 const double* gate, const double* maxa, const double* denom, double* dq,
                 double* dk, double* dv, double* gu);

#ifdef __cplusplus
}
#endif
#endif
