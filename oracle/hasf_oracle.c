/*
 * CPU oracle for the HASF path -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithm (toposmooth, pure Python +
 * numba) so that parity tests and the bench's cpu_baseline / --impl reference
 * arm can run without /root/reference.  Only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline leg and --impl reference) may load this library;
 * the product path (paper_1603_09337_b200) never does.
 *
 * Pinned against golden vectors generated from the imported reference
 * (tests/golden/make_golden.py -> tests/golden/ fixtures, checked by
 * tests/test_oracle_golden.py).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/toposmooth/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* edt.py:25-28 */
static int64_t inf_value(int64_t h, int64_t w) { return h * h + w * w + 1; }

/* Python floor division for a positive divisor (edt.py:42, edt.py:106). */
static int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

/* edt.py:31-42 (argument checks are done by the Python wrapper) */
int64_t orc_sep(int64_t i, int64_t u, int64_t gi, int64_t gu) {
    return floordiv(u * u - i * i + gu * gu - gi * gi, 2 * (u - i));
}

/* edt.py:45-71: column sweeps.  Seed = (pix != invert). */
static void phase1(const uint8_t *pix, int64_t *g, int h, int w, int64_t inf, int invert) {
    for (int c = 0; c < w; ++c) g[c] = (pix[c] != invert) ? 0 : inf;
    for (int r = 1; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            int64_t i = (int64_t)r * w + c;
            if (pix[i] != invert) g[i] = 0;
            else if (g[i - w] < inf) g[i] = g[i - w] + 1;
            else g[i] = inf;
        }
    for (int r = h - 2; r >= 0; --r)
        for (int c = 0; c < w; ++c) {
            int64_t i = (int64_t)r * w + c;
            if (g[i + w] < g[i]) g[i] = g[i + w] + 1;
        }
}

/* edt.py:74-119: per-row lower envelope of parabolas (Meijster phase 2). */
static void phase2(const int64_t *g, int64_t *out, int h, int m, int64_t inf,
                   int64_t *s, int64_t *t) {
    for (int r = 0; r < h; ++r) {
        const int64_t *gr = g + (int64_t)r * m;
        int64_t *orow = out + (int64_t)r * m;
        int64_t q = -1;
        for (int64_t u = 0; u < m; ++u) {
            int64_t gu = gr[u];
            if (gu >= inf) continue;
            if (q < 0) { q = 0; s[0] = u; t[0] = 0; continue; }
            while (q >= 0) {
                int64_t tq = t[q], sq = s[q];
                int64_t f_old = (tq - sq) * (tq - sq) + gr[sq] * gr[sq];
                int64_t f_new = (tq - u) * (tq - u) + gu * gu;
                if (f_old > f_new) q -= 1; else break;
            }
            if (q < 0) { q = 0; s[0] = u; t[0] = 0; }
            else {
                int64_t sq = s[q];
                int64_t wv = 1 + floordiv(u * u - sq * sq + gu * gu - gr[sq] * gr[sq], 2 * (u - sq));
                if (wv < m) { q += 1; s[q] = u; t[q] = wv; }
            }
        }
        if (q < 0) {
            for (int u = 0; u < m; ++u) orow[u] = inf;
        } else {
            for (int64_t u = m - 1; u >= 0; --u) {
                int64_t d = u - s[q];
                orow[u] = d * d + gr[s[q]] * gr[s[q]];
                if (u == t[q]) q -= 1;
            }
        }
    }
}

/* edt.py:152-170 (_edt_prepared); edt_squared's empty short-cut (edt.py:185-186)
 * gives the same INF fill, so one routine serves both. */
void orc_edt(const uint8_t *pix, int64_t *out, int h, int w, int invert) {
    int64_t inf = inf_value(h, w);
    int64_t *g = (int64_t *)malloc(sizeof(int64_t) * (size_t)h * w);
    int64_t *s = (int64_t *)malloc(sizeof(int64_t) * (size_t)w);
    int64_t *t = (int64_t *)malloc(sizeof(int64_t) * (size_t)w);
    phase1(pix, g, h, w, inf, invert);
    phase2(g, out, h, w, inf, s, t);
    free(g); free(s); free(t);
}

void orc_edt_phase1(const uint8_t *pix, int64_t *g, int h, int w) {
    phase1(pix, g, h, w, inf_value(h, w), 0);
}

void orc_edt_phase2(const int64_t *g, int64_t *out, int h, int w) {
    int64_t *s = (int64_t *)malloc(sizeof(int64_t) * (size_t)w);
    int64_t *t = (int64_t *)malloc(sizeof(int64_t) * (size_t)w);
    phase2(g, out, h, w, inf_value(h, w), s, t);
    free(s); free(t);
}

/* ---- simple-point LUT (topo.py:35-88) ---------------------------------- */
static const int OFF_R[8] = {-1, -1, -1, 0, 0, 1, 1, 1};   /* topo.py:35 */
static const int OFF_C[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
static uint8_t T8[256], T4[256], S84[256], S48[256];
static int lut_ready = 0;
static pthread_mutex_t lut_mu = PTHREAD_MUTEX_INITIALIZER;

/* topo.py:44-76: components of the set bits under conn, counting only those
 * conn-adjacent to the centre (all bits are 8-adjacent to it). */
static int count_components(int mask, int conn) {
    int seen = 0, count = 0;
    for (int start = 0; start < 8; ++start) {
        if (!((mask >> start) & 1) || ((seen >> start) & 1)) continue;
        int comp = 0, stack[8], sp = 0;
        stack[sp++] = start;
        while (sp) {
            int a = stack[--sp];
            if ((comp >> a) & 1) continue;
            comp |= 1 << a;
            for (int b = 0; b < 8; ++b) {
                if (!((mask >> b) & 1) || ((comp >> b) & 1)) continue;
                int dr = abs(OFF_R[a] - OFF_R[b]), dc = abs(OFF_C[a] - OFF_C[b]);
                int adjacent = (conn == 4) ? (dr + dc == 1) : ((dr > dc ? dr : dc) == 1);
                if (adjacent) stack[sp++] = b;
            }
        }
        seen |= comp;
        /* _EDGE_BITS = {1,3,4,6} (topo.py:36) */
        if (conn == 8 || (comp & ((1 << 1) | (1 << 3) | (1 << 4) | (1 << 6)))) count += 1;
    }
    return count;
}

static void build_luts(void) {
    pthread_mutex_lock(&lut_mu);
    if (!lut_ready) {
        for (int m = 0; m < 256; ++m) { T8[m] = count_components(m, 8); T4[m] = count_components(m, 4); }
        for (int m = 0; m < 256; ++m) {       /* topo.py:82-84 */
            S84[m] = (T8[m] == 1) && (T4[m ^ 0xFF] == 1);
            S48[m] = (T4[m] == 1) && (T8[m ^ 0xFF] == 1);
        }
        lut_ready = 1;
    }
    pthread_mutex_unlock(&lut_mu);
}

void orc_luts(uint8_t *t8, uint8_t *t4, uint8_t *s84, uint8_t *s48) {
    build_luts();
    memcpy(t8, T8, 256); memcpy(t4, T4, 256); memcpy(s84, S84, 256); memcpy(s48, S48, 256);
}

static const uint8_t *simple_lut(int fg) { build_luts(); return fg == 8 ? S84 : S48; }  /* topo.py:87-88 */

/* code of (r,c) from a zero-padded (h+2)x(w+2) frame (topo.py:196-203) */
static inline uint8_t padded_code(const uint8_t *pd, int wp, int r, int c) {
    int pr = r + 1, pc = c + 1;
    const uint8_t *u = pd + (int64_t)(pr - 1) * wp, *m = pd + (int64_t)pr * wp, *d = pd + (int64_t)(pr + 1) * wp;
    return (uint8_t)(u[pc - 1] | (u[pc] << 1) | (u[pc + 1] << 2) | (m[pc - 1] << 3) |
                     (m[pc + 1] << 4) | (d[pc - 1] << 5) | (d[pc] << 6) | (d[pc + 1] << 7));
}

/* ---- binary heap on packed keys (topo.py:151-183) ---------------------- */
static int64_t heap_push(int64_t *heap, int64_t n, int64_t key) {
    heap[n] = key;
    int64_t j = n;
    while (j > 0) {
        int64_t parent = (j - 1) >> 1;
        if (heap[parent] > heap[j]) { int64_t tmp = heap[parent]; heap[parent] = heap[j]; heap[j] = tmp; j = parent; }
        else break;
    }
    return n + 1;
}

static int64_t heap_pop(int64_t *heap, int64_t n, int64_t *key) {
    *key = heap[0];
    n -= 1;
    heap[0] = heap[n];
    int64_t j = 0;
    for (;;) {
        int64_t left = 2 * j + 1, right = left + 1, best = j;
        if (left < n && heap[left] < heap[best]) best = left;
        if (right < n && heap[right] < heap[best]) best = right;
        if (best == j) break;
        int64_t tmp = heap[best]; heap[best] = heap[j]; heap[j] = tmp;
        j = best;
    }
    return n;
}

/* topo.py:211-258: sequential priority-ordered removal.  Returns the number of
 * sweeps executed (instrumentation only). */
static int64_t thin_engine(uint8_t *pix, uint8_t *code, const uint8_t *blocked,
                           const int64_t *priority, const uint8_t *lut,
                           const uint8_t *cand, int h, int w, int64_t max_sweeps) {
    int64_t nm = (int64_t)h * w;
    int64_t *heap = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nm ? nm : 1));
    uint8_t *in_heap = (uint8_t *)calloc((size_t)(nm ? nm : 1), 1);
    int64_t *touched = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nm ? nm : 1));
    int64_t hn = 0;
    for (int64_t idx = 0; idx < nm; ++idx)           /* np.flatnonzero(cand) order */
        if (cand[idx]) { hn = heap_push(heap, hn, priority[idx] * nm + idx); in_heap[idx] = 1; }
    int64_t sweeps = 0;
    while (hn > 0 && (max_sweeps < 0 || sweeps < max_sweeps)) {
        int64_t top = 0;
        while (hn > 0) {
            int64_t key;
            hn = heap_pop(heap, hn, &key);
            int64_t idx = key % nm;
            in_heap[idx] = 0;
            int r = (int)(idx / w), c = (int)(idx - (int64_t)r * w);
            if (pix[idx] == 1 && blocked[idx] == 0 && lut[code[idx]] == 1) {
                pix[idx] = 0;
                for (int k = 0; k < 8; ++k) {
                    int nr = r + OFF_R[k], nc = c + OFF_C[k];
                    if (nr >= 0 && nr < h && nc >= 0 && nc < w)
                        code[(int64_t)nr * w + nc] ^= (uint8_t)(1 << (7 - k));   /* _FLIP, topo.py:41 */
                }
                touched[top++] = idx;
            }
        }
        while (top > 0) {
            int64_t idx = touched[--top];
            int r = (int)(idx / w), c = (int)(idx - (int64_t)r * w);
            for (int k = 0; k < 8; ++k) {
                int nr = r + OFF_R[k], nc = c + OFF_C[k];
                if (nr >= 0 && nr < h && nc >= 0 && nc < w) {
                    int64_t nidx = (int64_t)nr * w + nc;
                    if (in_heap[nidx] == 0 && pix[nidx] == 1 && blocked[nidx] == 0 && lut[code[nidx]] == 1) {
                        hn = heap_push(heap, hn, priority[nidx] * nm + nidx);
                        in_heap[nidx] = 1;
                    }
                }
            }
        }
        sweeps += 1;
    }
    free(heap); free(in_heap); free(touched);
    return sweeps;
}

/* topo.py:279-300 (_thin_prepared): detect pass (topo.py:186-208) + engine. */
static int64_t thin_prepared(const uint8_t *pix, const uint8_t *keep, const int64_t *priority,
                             int fg, int64_t max_iter, uint8_t *out, int h, int w) {
    int64_t nm = (int64_t)h * w;
    int wp = w + 2;
    memcpy(out, pix, (size_t)nm);
    uint8_t *padded = (uint8_t *)calloc((size_t)(h + 2) * wp, 1);
    for (int r = 0; r < h; ++r) memcpy(padded + (int64_t)(r + 1) * wp + 1, out + (int64_t)r * w, (size_t)w);
    const uint8_t *lut = simple_lut(fg);
    uint8_t *code = (uint8_t *)malloc((size_t)(nm ? nm : 1));
    uint8_t *cand = (uint8_t *)malloc((size_t)(nm ? nm : 1));
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            int64_t i = (int64_t)r * w + c;
            uint8_t v = padded_code(padded, wp, r, c);
            code[i] = v;
            cand[i] = (padded[(int64_t)(r + 1) * wp + c + 1] == 1 && keep[i] == 0 && lut[v] == 1);
        }
    int64_t sweeps = thin_engine(out, code, keep, priority, lut, cand, h, w, max_iter);
    free(padded); free(code); free(cand);
    return sweeps;
}

/* topo.py:303-314 (validation in Python) */
int64_t orc_homotopic_thin(const uint8_t *pix, const uint8_t *keep, const int64_t *priority,
                           int fg, int64_t max_iter, uint8_t *out, int h, int w) {
    return thin_prepared(pix, keep, priority, fg, max_iter, out, h, w);
}

/* topo.py:345-354: thicken = thin the ring-padded complement under adj.dual(). */
static int64_t thicken_prepared(const uint8_t *pix, const uint8_t *allowed, const int64_t *priority,
                                int fg, int64_t max_iter, uint8_t *out, int h, int w) {
    int hp = h + 2, wp = w + 2;
    size_t np_ = (size_t)hp * wp;
    uint8_t *z = (uint8_t *)malloc(np_), *floor_ = (uint8_t *)malloc(np_), *th = (uint8_t *)malloc(np_);
    int64_t *prio = (int64_t *)calloc(np_, sizeof(int64_t));
    memset(z, 1, np_); memset(floor_, 1, np_);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            int64_t i = (int64_t)r * w + c, j = (int64_t)(r + 1) * wp + c + 1;
            z[j] = pix[i] ^ 1;
            floor_[j] = allowed[i] ^ 1;
            prio[j] = priority[i];
        }
    int dual = 12 - fg;                               /* grid.py:34-41 */
    int64_t sweeps = thin_prepared(z, floor_, prio, dual, max_iter, th, hp, wp);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) out[(int64_t)r * w + c] = th[(int64_t)(r + 1) * wp + c + 1] ^ 1;
    free(z); free(floor_); free(th); free(prio);
    return sweeps;
}

int64_t orc_homotopic_thicken(const uint8_t *pix, const uint8_t *allowed, const int64_t *priority,
                              int fg, int64_t max_iter, uint8_t *out, int h, int w) {
    return thicken_prepared(pix, allowed, priority, fg, max_iter, out, h, w);
}

/* smoothing.py:107-124 (_constrained_thin) with the fused prepare kernel
 * smoothing.py:51-86. */
static void constrained_thin(const uint8_t *pix, const uint8_t *keep, int64_t rsq, int fg,
                             uint8_t *out, int h, int w) {
    int64_t nm = (int64_t)h * w;
    const uint8_t *lut = simple_lut(fg);
    int64_t *dist_bg = (int64_t *)malloc(sizeof(int64_t) * (size_t)nm);
    orc_edt(pix, dist_bg, h, w, 1);
    int wp = w + 2;
    uint8_t *padded = (uint8_t *)calloc((size_t)(h + 2) * wp, 1);
    for (int r = 0; r < h; ++r) memcpy(padded + (int64_t)(r + 1) * wp + 1, pix + (int64_t)r * w, (size_t)w);
    uint8_t *floor_ = (uint8_t *)malloc((size_t)nm), *code = (uint8_t *)malloc((size_t)nm),
            *cand = (uint8_t *)malloc((size_t)nm);
    int64_t *priority = (int64_t *)malloc(sizeof(int64_t) * (size_t)nm);
    for (int r = 0; r < h; ++r) {
        int64_t rb = (r + 1 < h - r) ? r + 1 : h - r;
        for (int c = 0; c < w; ++c) {
            int64_t i = (int64_t)r * w + c;
            int64_t cb = (c + 1 < w - c) ? c + 1 : w - c;
            int64_t b = rb < cb ? rb : cb;
            int64_t p = dist_bg[i];
            if (b * b < p) p = b * b;
            priority[i] = p;
            uint8_t blocked = (p > rsq || keep[i] == 1) ? 1 : 0;
            floor_[i] = blocked;
            uint8_t v = padded_code(padded, wp, r, c);
            code[i] = v;
            cand[i] = (padded[(int64_t)(r + 1) * wp + c + 1] == 1 && blocked == 0 && lut[v] == 1);
        }
    }
    memcpy(out, pix, (size_t)nm);
    thin_engine(out, code, floor_, priority, lut, cand, h, w, -1);
    free(dist_bg); free(padded); free(floor_); free(code); free(cand); free(priority);
}

/* smoothing.py:127-135 */
void orc_cutting(const uint8_t *pix, const uint8_t *keep, int r, int fg, uint8_t *out, int h, int w) {
    int64_t nm = (int64_t)h * w, rsq = (int64_t)r * r;
    uint8_t *thinned = (uint8_t *)malloc((size_t)nm), *cap = (uint8_t *)malloc((size_t)nm);
    int64_t *dist_y = (int64_t *)malloc(sizeof(int64_t) * (size_t)nm);
    constrained_thin(pix, keep, rsq, fg, thinned, h, w);
    orc_edt(thinned, dist_y, h, w, 0);
    for (int64_t i = 0; i < nm; ++i) cap[i] = (dist_y[i] <= rsq && pix[i] == 1);   /* smoothing.py:89-100 */
    thicken_prepared(thinned, cap, dist_y, fg, -1, out, h, w);
    free(thinned); free(cap); free(dist_y);
}

/* smoothing.py:138-146 */
void orc_filling(const uint8_t *pix, const uint8_t *avoid, int r, int fg, uint8_t *out, int h, int w) {
    int64_t nm = (int64_t)h * w, rsq = (int64_t)r * r;
    uint8_t *thick = (uint8_t *)malloc((size_t)nm), *cap = (uint8_t *)malloc((size_t)nm);
    int64_t *dist_x = (int64_t *)malloc(sizeof(int64_t) * (size_t)nm);
    orc_edt(pix, dist_x, h, w, 0);
    for (int64_t i = 0; i < nm; ++i) cap[i] = (dist_x[i] <= rsq && avoid[i] == 0);
    thicken_prepared(pix, cap, dist_x, fg, -1, thick, h, w);
    constrained_thin(thick, pix, rsq, fg, out, h, w);
    free(thick); free(cap); free(dist_x);
}

/* smoothing.py:187-212 (validation in Python).  keep/avoid may be NULL. */
void orc_hasf(const uint8_t *pix, const uint8_t *keep, const uint8_t *avoid, int r_max, int fg,
              uint8_t *out, int h, int w) {
    int64_t nm = (int64_t)h * w;
    uint8_t *zeros = NULL;
    if (!keep || !avoid) {
        zeros = (uint8_t *)calloc((size_t)nm, 1);
        if (!keep) keep = zeros;
        if (!avoid) avoid = zeros;
    }
    uint8_t *cur = (uint8_t *)malloc((size_t)nm), *tmp = (uint8_t *)malloc((size_t)nm);
    memcpy(cur, pix, (size_t)nm);
    for (int r = 1; r <= r_max; ++r) {
        orc_cutting(cur, keep, r, fg, tmp, h, w);
        orc_filling(tmp, avoid, r, fg, cur, h, w);
    }
    memcpy(out, cur, (size_t)nm);
    free(cur); free(tmp); free(zeros);
}

/* Batch driver: independent images over a pthread pool (images are the unit of
 * parallelism; the engine holds no shared state).  keep/avoid may be NULL or
 * [n,h,w]. */
typedef struct {
    const uint8_t *in, *keep, *avoid; uint8_t *out;
    int64_t n; int h, w, r_max, fg;
    int64_t next; pthread_mutex_t mu;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *j = (batch_job *)arg;
    int64_t nm = (int64_t)j->h * j->w;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int64_t i = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->n) break;
        orc_hasf(j->in + i * nm, j->keep ? j->keep + i * nm : NULL, j->avoid ? j->avoid + i * nm : NULL,
                 j->r_max, j->fg, j->out + i * nm, j->h, j->w);
    }
    return NULL;
}

void orc_hasf_batch(const uint8_t *in, const uint8_t *keep, const uint8_t *avoid, int64_t n, int h, int w,
                    int r_max, int fg, uint8_t *out, int threads) {
    build_luts();
    batch_job j = {in, keep, avoid, out, n, h, w, r_max, fg, 0, PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = 1;
    if (threads > 1024) threads = 1024;
    pthread_t tid[1024];
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, batch_worker, &j);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}
