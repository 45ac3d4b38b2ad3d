/* TEST INFRASTRUCTURE ONLY — CPU oracle restating the reference algorithm.
 * See sparsek_oracle.h. Citations are relative to /root/reference/. */
#include "sparsek_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_SHAPE 1
#define ORC_ARG 2
#define ORC_NUMERIC 3

static const double NEG_INF = -INFINITY;

/* ---------------------------------------------------------------- scoring */

/* proj/include/sparsek/selection.hpp:69-96; Welford push proj/src/selection.cpp:13-20. */
int orc_score_fwd(const double* x, const double* w, int64_t L, int64_t D, int32_t norm_mode,
                  int32_t slope_order, int32_t slope_enabled, double slope_eps, double* raw,
                  double* u, double* mean, double* sdev) {
    int64_t count = 0;
    double mu = 0.0, m2 = 0.0;
    const double eps = 1e-5;
    for (int64_t i = 0; i < L; ++i) {
        double r = 0.0;
        for (int64_t c = 0; c < D; ++c) r += x[i * D + c] * w[c];
        if (!isfinite(r)) return ORC_NUMERIC;
        const double slope = slope_enabled ? (double)(i + 1) * slope_eps : 0.0;
        if (norm_mode == 0) {
            raw[i] = r;
            u[i] = r + slope;
            mean[i] = 0.0;
            sdev[i] = 1.0;
            continue;
        }
        const double rin = slope_order == 0 ? r + slope : r;
        ++count;
        const double delta = rin - mu;
        mu += delta / (double)count;
        m2 += delta * (rin - mu);
        const double var = m2 / (double)count;
        const double z = (rin - mu) / sqrt(var + eps);
        raw[i] = rin;
        u[i] = slope_order == 0 ? z : z + slope;
        mean[i] = mu;
        sdev[i] = sqrt(var + eps);
    }
    return ORC_OK;
}

/* proj/src/attention.cpp:482-502 (single chunk: cs_of[j] = 0). */
void orc_score_bwd(const double* gu, const double* raw, const double* mean, const double* sdev,
                   int64_t L, int32_t norm_mode, double* graw) {
    for (int64_t j = 0; j < L; ++j) graw[j] = 0.0;
    if (norm_mode == 0) {
        for (int64_t j = 0; j < L; ++j) graw[j] = gu[j];
        return;
    }
    for (int64_t j = 0; j < L; ++j) {
        if (gu[j] == 0.0) continue;
        const double cnt = (double)(j + 1);
        const double s = sdev[j], mu = mean[j];
        const double yj = (raw[j] - mu) / s;
        const double coef = gu[j] / s;
        for (int64_t j2 = 0; j2 <= j; ++j2) {
            const double delta = j2 == j ? 1.0 : 0.0;
            graw[j2] += coef * (delta - 1.0 / cnt - yj * (raw[j2] - mu) / (cnt * s));
        }
    }
}

/* --------------------------------------------------------- batch SparseK */

static int cmp_desc(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

/* scan_sorted, proj/src/sparsek_op.cpp:63-98 (exact mode). */
static int scan_sorted(const double* zs, int64_t c, double k, double* tau_out) {
    double* csum = (double*)malloc(sizeof(double) * (size_t)(c + 1));
    if (!csum) return ORC_NUMERIC;
    csum[0] = 0.0;
    for (int64_t i = 0; i < c; ++i) csum[i + 1] = csum[i] + zs[i];
    int64_t u = c, w = c;
    int rc = ORC_OK;
    for (;;) {
        if (u == w) {
            const int budget_hits = fabs((double)u - k) <= 1e-9;
            const double hi = zs[u - 1] - 1.0;
            const double lo = (u < c) ? zs[u] : hi - 1.0;
            if (budget_hits && lo <= hi) {
                *tau_out = 0.5 * (lo + hi);
                break;
            }
            --u;
            continue;
        }
        const double tau = (csum[w] - csum[u] + (double)u - k) / (double)(w - u);
        if (zs[w - 1] > tau && (u == 0 || zs[u - 1] >= tau + 1.0)) {
            *tau_out = tau;
            break;
        }
        if (u == 0 || zs[w - 1] <= zs[u - 1] - 1.0) {
            --w;
            if (w == 0) {
                rc = ORC_NUMERIC;
                break;
            }
        } else {
            --u;
        }
    }
    free(csum);
    return rc;
}

/* sparsek + finish, proj/src/sparsek_op.cpp:36-57, 102-114. */
int orc_sparsek(const double* z, int64_t m, double k, double* p, double* tau, int64_t* u_count,
                int64_t* w_count, int32_t* degenerate, int32_t* infeasible) {
    if (m <= 0) return ORC_ARG;
    if (!(k > 0.0) || !isfinite(k)) return ORC_ARG;
    for (int64_t i = 0; i < m; ++i)
        if (!isfinite(z[i])) return ORC_NUMERIC;
    if (k > (double)m) { /* all_ones, sparsek_op.cpp:21-32 */
        for (int64_t i = 0; i < m; ++i) p[i] = 1.0;
        *tau = NEG_INF;
        *u_count = m;
        *w_count = m;
        *degenerate = 1;
        *infeasible = 1;
        return ORC_OK;
    }
    double* zs = (double*)malloc(sizeof(double) * (size_t)m);
    memcpy(zs, z, sizeof(double) * (size_t)m);
    qsort(zs, (size_t)m, sizeof(double), cmp_desc);
    double t = 0.0;
    int rc = scan_sorted(zs, m, k, &t);
    free(zs);
    if (rc) return rc;
    *tau = t;
    int64_t uc = 0, wc = 0, sup = 0;
    for (int64_t j = 0; j < m; ++j) {
        double pj = z[j] - t;
        pj = pj < 0.0 ? 0.0 : (pj > 1.0 ? 1.0 : pj);
        p[j] = pj;
        if (pj == 1.0) {
            ++uc;
            ++wc;
        } else if (pj > 0.0) {
            ++wc;
            ++sup;
        }
    }
    *u_count = uc;
    *w_count = wc;
    *degenerate = sup == 0;
    *infeasible = 0;
    return ORC_OK;
}

/* proj/src/sparsek_op.cpp:141-150 */
int orc_sparsek_jvp(const double* z, int64_t m, double k, const double* v, double* out) {
    double* p = (double*)malloc(sizeof(double) * (size_t)m);
    double tau;
    int64_t uc, wc;
    int32_t deg, inf;
    int rc = orc_sparsek(z, m, k, p, &tau, &uc, &wc, &deg, &inf);
    if (rc) {
        free(p);
        return rc;
    }
    double acc = 0.0;
    int64_t n = 0;
    for (int64_t j = 0; j < m; ++j)
        if (p[j] > 0.0 && p[j] < 1.0) {
            acc += v[j];
            ++n;
        }
    for (int64_t j = 0; j < m; ++j) out[j] = 0.0;
    if (n) {
        const double vbar = acc / (double)n;
        for (int64_t j = 0; j < m; ++j)
            if (p[j] > 0.0 && p[j] < 1.0) out[j] = v[j] - vbar;
    }
    free(p);
    return ORC_OK;
}

/* proj/src/sparsek_op.cpp:152-165: k largest, ties to the lower index. */
void orc_topk_hard(const double* z, int64_t m, int64_t k, double* out) {
    for (int64_t i = 0; i < m; ++i) out[i] = 0.0;
    if (k >= m) {
        for (int64_t i = 0; i < m; ++i) out[i] = 1.0;
        return;
    }
    for (int64_t i = 0; i < m; ++i) {
        int64_t better = 0; /* entries ranked ahead of i */
        for (int64_t j = 0; j < m && better < k; ++j)
            if (z[j] > z[i] || (z[j] == z[i] && j < i)) ++better;
        if (better < k) out[i] = 1.0;
    }
}

/* -------------------------------------------------------------- the stream */

/* Min-heap with the reference's HeapCmp (proj/src/stream.cpp:14-18) and
 * SlotCmp (proj/src/cache.cpp:53-60): front = lowest value, ties -> larger index. */
typedef struct {
    double v;
    int64_t i;
} orc_ent;
typedef struct {
    orc_ent* a;
    int64_t n, cap;
} orc_heap;

static int ent_above(orc_ent x, orc_ent y) { /* x nearer the front than y */
    return x.v < y.v || (x.v == y.v && x.i > y.i);
}
static void heap_push(orc_heap* h, orc_ent e) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->a = (orc_ent*)realloc(h->a, sizeof(orc_ent) * (size_t)h->cap);
    }
    int64_t c = h->n++;
    h->a[c] = e;
    while (c > 0) {
        int64_t par = (c - 1) / 2;
        if (!ent_above(h->a[c], h->a[par])) break;
        orc_ent t = h->a[c];
        h->a[c] = h->a[par];
        h->a[par] = t;
        c = par;
    }
}
static orc_ent heap_pop(orc_heap* h) {
    orc_ent top = h->a[0];
    h->a[0] = h->a[--h->n];
    int64_t c = 0;
    for (;;) {
        int64_t l = 2 * c + 1, r = l + 1, b = c;
        if (l < h->n && ent_above(h->a[l], h->a[b])) b = l;
        if (r < h->n && ent_above(h->a[r], h->a[b])) b = r;
        if (b == c) break;
        orc_ent t = h->a[c];
        h->a[c] = h->a[b];
        h->a[b] = t;
        c = b;
    }
    return top;
}

typedef struct {
    double k, tau, sum_s, sum_f;
    int64_t t;
    orc_heap S, F;
} orc_stream;

/* StreamState::push, proj/src/stream.cpp:72-152 (unbounded heaps; the 2^16
 * sum refresh at :78-81 is not restated — callers stay below 65536 pushes). */
static int stream_push(orc_stream* st, double z, double* tau_out, int* inserted) {
    if (!isfinite(z)) return ORC_NUMERIC;
    st->t++;
    *inserted = 0;
    if (!(z > st->tau)) {
        *tau_out = st->tau;
        return ORC_OK;
    }
    *inserted = 1;
    orc_ent e = {z, st->t - 1};
    heap_push(&st->S, e);
    st->sum_s += z;
    if (z >= st->tau + 1.0) {
        heap_push(&st->F, e);
        st->sum_f += z;
    }
    if ((double)st->t < st->k) {
        *tau_out = NEG_INF;
        return ORC_OK;
    }
    int popped = 0;
    double last = 0.0;
    for (;;) {
        const int64_t u = st->F.n, w = st->S.n;
        if (u == w) {
            const double hi = st->F.a[0].v - 1.0;
            const double lo = popped ? last : fmax(st->tau, hi - 1.0);
            if (fabs((double)u - st->k) <= 1e-9) {
                st->tau = fmax(st->tau, 0.5 * (lo + hi));
                break;
            }
            st->sum_f -= heap_pop(&st->F).v;
            continue;
        }
        const double cand = (st->sum_s - st->sum_f + (double)u - st->k) / (double)(w - u);
        if (st->S.a[0].v > cand && (u == 0 || st->F.a[0].v >= cand + 1.0)) {
            st->tau = cand;
            break;
        }
        if (u == 0 || st->S.a[0].v <= st->F.a[0].v - 1.0) {
            last = st->S.a[0].v;
            popped = 1;
            st->sum_s -= heap_pop(&st->S).v;
            if (st->S.n == 0) return ORC_NUMERIC;
        } else {
            st->sum_f -= heap_pop(&st->F).v;
        }
    }
    *tau_out = st->tau;
    return ORC_OK;
}

static void stream_free(orc_stream* st) {
    free(st->S.a);
    free(st->F.a);
}

int orc_stream_taus(const double* z, int64_t n, double k, double* tau_out, uint8_t* inserted) {
    if (!(k > 0.0) || !isfinite(k)) return ORC_ARG;
    orc_stream st;
    memset(&st, 0, sizeof st);
    st.k = k;
    st.tau = NEG_INF;
    for (int64_t t = 0; t < n; ++t) {
        int ins = 0;
        int rc = stream_push(&st, z[t], &tau_out[t], &ins);
        if (rc) {
            stream_free(&st);
            return rc;
        }
        if (inserted) inserted[t] = (uint8_t)ins;
    }
    stream_free(&st);
    return ORC_OK;
}

/* ------------------------------------------------- retention + snapshots */

/* SparseKvCache::exit_window / admit_to_cache (proj/src/cache.cpp:136-179) and
 * the per-query snapshot (proj/src/cache.cpp:259-311). */
int orc_select(const double* u, int64_t L, double k, int64_t window, double* tau_q,
               int32_t* n_sel, int64_t* att_off, int32_t* att, double* gate) {
    if (!(k >= 0.0) || !isfinite(k) || window < 0) return ORC_ARG;
    if (window == 0 && floor(k) < 1.0) return ORC_ARG; /* attention.cpp:27-31 */
    const int64_t cap = k > 0.0 ? (int64_t)floor(k) : 0;
    orc_stream st;
    memset(&st, 0, sizeof st);
    st.k = k;
    st.tau = NEG_INF;
    orc_heap cache = {0, 0, 0};
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap + 1)); /* sorted retained */
    int64_t npos = 0;
    int64_t off = 0;
    int rc = ORC_OK;
    for (int64_t i = 0; i < L; ++i) {
        /* ring holds [max(0,i-w+1), i] after the exit of i-w */
        const int64_t exiting = i - window;
        if (exiting >= 0) {
            int admitted = 0;
            if (k > 0.0) {
                double tau;
                int ins;
                rc = stream_push(&st, u[exiting], &tau, &ins);
                if (rc) goto done;
                if (ins && cap > 0) {
                    const double s = u[exiting];
                    if (cache.n < cap) {
                        orc_ent e = {s, exiting};
                        heap_push(&cache, e);
                        pos[npos++] = exiting;
                        admitted = 1;
                    } else {
                        const orc_ent worst = cache.a[0];
                        if (!(s < worst.v || s == worst.v)) {
                            heap_pop(&cache);
                            orc_ent e = {s, exiting};
                            heap_push(&cache, e);
                            int64_t a = 0;
                            while (pos[a] != worst.i) ++a;
                            memmove(pos + a, pos + a + 1, sizeof(int64_t) * (size_t)(npos - a - 1));
                            pos[npos - 1] = exiting;
                            admitted = 1;
                        }
                    }
                }
            }
            (void)admitted;
        }
        tau_q[i] = (exiting >= 0 && k > 0.0) ? st.tau : NEG_INF;
        n_sel[i] = (int32_t)npos;
        const int64_t wlo = i - window + 1 > 0 ? i - window + 1 : 0;
        int64_t n = npos + (i - wlo + 1);
        int self = 0;
        if (window == 0) {
            const int selected = npos > 0 && pos[npos - 1] == i;
            if (!selected) self = 1;
            n = npos + self;
        }
        att_off[i] = off;
        if (att) {
            for (int64_t a = 0; a < npos; ++a) {
                att[off + a] = (int32_t)pos[a];
                double g = u[pos[a]] - st.tau;
                g = g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g); /* cache.cpp:293 */
                gate[off + a] = g;
            }
            int64_t a = npos;
            if (window > 0)
                for (int64_t r = wlo; r <= i; ++r, ++a) {
                    att[off + a] = (int32_t)r;
                    gate[off + a] = 1.0;
                }
            if (self) {
                att[off + a] = (int32_t)i;
                gate[off + a] = 1.0;
            }
        }
        off += n;
    }
    att_off[L] = off;
done:
    free(pos);
    free(cache.a);
    stream_free(&st);
    return rc;
}

/* -------------------------------------------------------------- attention */

static double eff_scale(const orc_cfg* c, int64_t p) {
    return c->scale > 0.0 ? c->scale : 1.0 / sqrt((double)p);
}

/* proj/src/cache.cpp:358-393 */
int orc_attn_fwd(const double* q, const double* k, const double* v, int64_t L, int64_t p,
                 const orc_cfg* cfg, const int32_t* n_sel, const int64_t* att_off,
                 const int32_t* att, const double* gate, double* o, double* maxa, double* denom) {
    const int64_t H = cfg->heads, D = H * p;
    const double scale = eff_scale(cfg, p);
    int64_t maxn = 0;
    for (int64_t i = 0; i < L; ++i)
        if (att_off[i + 1] - att_off[i] > maxn) maxn = att_off[i + 1] - att_off[i];
    double* a = (double*)malloc(sizeof(double) * (size_t)(maxn + 1));
    for (int64_t i = 0; i < L; ++i) {
        const int64_t base = att_off[i], n = att_off[i + 1] - base;
        for (int64_t h = 0; h < H; ++h) {
            const double* qi = q + i * D + h * p;
            double* oi = o + i * D + h * p;
            for (int64_t c = 0; c < p; ++c) oi[c] = 0.0;
            double mx = -INFINITY;
            for (int64_t jd = 0; jd < n; ++jd) {
                const double* kj = k + (int64_t)att[base + jd] * D + h * p;
                double dot = 0.0;
                for (int64_t c = 0; c < p; ++c) dot += qi[c] * kj[c];
                double aj = scale * dot;
                if (cfg->key_soft && jd < n_sel[i]) aj *= gate[base + jd];
                a[jd] = aj;
                if (aj > mx) mx = aj;
            }
            double den = 0.0;
            for (int64_t jd = 0; jd < n; ++jd) {
                a[jd] = exp(a[jd] - mx);
                den += a[jd];
            }
            for (int64_t jd = 0; jd < n; ++jd) {
                const double pi = a[jd] / den;
                const double wv = (jd < n_sel[i] && !cfg->mask_st) ? gate[base + jd] : 1.0;
                const double* vj = v + (int64_t)att[base + jd] * D + h * p;
                const double c0 = pi * wv;
                for (int64_t c = 0; c < p; ++c) oi[c] += c0 * vj[c];
            }
            maxa[i * H + h] = mx;
            denom[i * H + h] = den;
        }
    }
    free(a);
    return ORC_OK;
}

/* proj/src/attention.cpp:259-316 (softmax/gate backward, non-linear-mix) and
 * :447-479 (selection pullback over the full fractional support). */
int orc_attn_bwd(const double* q, const double* k, const double* v, const double* dout,
                 int64_t L, int64_t p, const orc_cfg* cfg, const double* u, const double* tau_q,
                 const int32_t* n_sel, const int64_t* att_off, const int32_t* att,
                 const double* gate, const double* maxa, const double* denom, double* dq,
                 double* dk, double* dv, double* gu) {
    const int64_t H = cfg->heads, D = H * p, w = cfg->window;
    const double scale = eff_scale(cfg, p);
    memset(dq, 0, sizeof(double) * (size_t)(L * D));
    memset(dk, 0, sizeof(double) * (size_t)(L * D));
    memset(dv, 0, sizeof(double) * (size_t)(L * D));
    memset(gu, 0, sizeof(double) * (size_t)L);
    int64_t maxn = 0;
    for (int64_t i = 0; i < L; ++i)
        if (att_off[i + 1] - att_off[i] > maxn) maxn = att_off[i + 1] - att_off[i];
    double* pis = (double*)malloc(sizeof(double) * (size_t)(maxn + 1));
    double* bws = (double*)malloc(sizeof(double) * (size_t)(maxn + 1));
    double* gm = (double*)malloc(sizeof(double) * (size_t)(maxn + 1));
    for (int64_t i = 0; i < L; ++i) {
        const int64_t base = att_off[i], n = att_off[i + 1] - base, ns = n_sel[i];
        for (int64_t jd = 0; jd < ns; ++jd) gm[jd] = 0.0;
        for (int64_t h = 0; h < H; ++h) {
            const double* qi = q + i * D + h * p;
            const double* gi = dout + i * D + h * p;
            const double mx = maxa[i * H + h], den = denom[i * H + h];
            double s = 0.0;
            for (int64_t jd = 0; jd < n; ++jd) {
                const int64_t j = att[base + jd];
                const double* kj = k + j * D + h * p;
                const double* vj = v + j * D + h * p;
                double dot = 0.0;
                for (int64_t c = 0; c < p; ++c) dot += qi[c] * kj[c];
                double aj = scale * dot;
                if (cfg->key_soft && jd < ns) aj *= gate[base + jd];
                const double pi = exp(aj - mx) / den;
                const double wv = (jd < ns && !cfg->mask_st) ? gate[base + jd] : 1.0;
                double b = 0.0;
                for (int64_t c = 0; c < p; ++c) b += gi[c] * vj[c];
                pis[jd] = pi;
                bws[jd] = wv * b;
                s += pi * wv * b;
                const double c0 = pi * wv;
                double* dvj = dv + j * D + h * p;
                for (int64_t c = 0; c < p; ++c) dvj[c] += c0 * gi[c];
                if (jd < ns) gm[jd] += pi * b;
            }
            for (int64_t jd = 0; jd < n; ++jd) {
                const int64_t j = att[base + jd];
                const double* kj = k + j * D + h * p;
                const double cj = pis[jd] * (bws[jd] - s);
                const int gated = cfg->key_soft && jd < ns;
                const double kap = gated ? gate[base + jd] : 1.0;
                const double coef = scale * cj * kap;
                double* dqi = dq + i * D + h * p;
                double* dkj = dk + j * D + h * p;
                for (int64_t c = 0; c < p; ++c) dqi[c] += coef * kj[c];
                for (int64_t c = 0; c < p; ++c) dkj[c] += coef * qi[c];
                if (gated) {
                    double dot = 0.0;
                    for (int64_t c = 0; c < p; ++c) dot += qi[c] * kj[c];
                    gm[jd] += scale * cj * dot;
                }
            }
        }
        if (ns) {
            const int64_t state_t = i - w;
            const double tau = tau_q[i];
            double gsum = 0.0;
            int64_t cnt = 0, sel = 0;
            for (int64_t j = 0; j <= state_t; ++j) {
                while (sel < ns && att[base + sel] < j) ++sel;
                const double f = u[j] - tau;
                if (f > 0.0 && f < 1.0) {
                    ++cnt;
                    if (sel < ns && att[base + sel] == j) gsum += gm[sel];
                }
            }
            if (cnt) {
                const double mean = gsum / (double)cnt;
                sel = 0;
                for (int64_t j = 0; j <= state_t; ++j) {
                    while (sel < ns && att[base + sel] < j) ++sel;
                    const double f = u[j] - tau;
                    if (f > 0.0 && f < 1.0) {
                        const double gmj = (sel < ns && att[base + sel] == j) ? gm[sel] : 0.0;
                        gu[j] += gmj - mean;
                    }
                }
            }
        }
    }
    free(pis);
    free(bws);
    free(gm);
    return ORC_OK;
}
