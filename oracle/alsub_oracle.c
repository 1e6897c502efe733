/*
 * alsub_oracle.c -- the CPU oracle: ONE uniform refinement level of Catmull-Clark, Loop or sqrt3,
 * written as the plain definition.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  It shares no code with paper_1809_06047_b200/.
 *
 * Deliberately naive: edges are found by sorting every slot's undirected key (hi, lo) with qsort
 * and looking slots up by rank; every per-vertex quantity is a loop over explicit incidence lists.
 * No blocking, fusion, structured shortcuts or reordering beyond the definitions.
 *
 * Parity pins: tests/test_oracle_pins.py (counts, Euler characteristic, hand values, B-spline
 * masks, affine invariance, crease limits, brute force vs exact rationals).  The paper gives no
 * numbers for the semi-sharp blend (0 < sigma < 1) or the >= 3-crease average (P:L411-413, L428,
 * L440); both are pinned by hand-derived values of readings R7/R8/R21 (tests/golden/
 * hand_values.json: cc_semisharp_vertex_L1, cc_three_creases_L1, cc_sigma_bar_exclusions_L1)
 * and by s -> 0+ / 1- continuity against the smooth and sharp hand values.
 */
#include "alsub_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* OpenMP appears only in the separately compiled liboracle_omp.so that times the oracle on all
 * host cores.  It marks the per-face / per-edge / per-vertex loops of a level,
 * each iteration the single writer of its outputs with no reductions, so the results are
 * identical to the serial build that the tests use.  The edge sort (qsort) stays serial. */
#ifdef _OPENMP
#include <omp.h>
#define OM_PARALLEL_FOR _Pragma("omp parallel for schedule(static)")
#else
#define OM_PARALLEL_FOR
#endif

int om_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* ------------------------------------------------------------------------------------------ */
static void set_err(char *err, int len, const char *fmt, ...) {
    if (!err || len <= 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, (size_t)len, fmt, ap);
    va_end(ap);
}

static void *xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz ? sz : 1); }

void om_mesh_free(om_mesh *m) {
    if (!m) return;
    free(m->face_off); free(m->face_vtx); free(m->pos); free(m->crease); free(m->sigma);
    memset(m, 0, sizeof(*m));
}

void om_edges_free(om_edges *e) {
    if (!e) return;
    free(e->edge_vtx); free(e->edge_face);
    memset(e, 0, sizeof(*e));
}

/* Loop's beta: beta_n = (1/n) (5/8 - (3/8 + 1/4 cos(2 pi / n))^2). */
double om_loop_beta(int n) {
    double c = 0.375 + 0.25 * cos(2.0 * M_PI / (double)n);
    return (0.625 - c * c) / (double)n;
}

/* sqrt3's alpha: alpha_n = (4 - 2 cos(2 pi / n)) / 9. */
double om_sqrt3_alpha(int n) { return (4.0 - 2.0 * cos(2.0 * M_PI / (double)n)) / 9.0; }

/* ------------------------------------------------------------------------------------------ */
/* Topology of one level: the mesh matrix M, the slot <-> edge correspondence behind
 * E = M M^T {Q_c + Q_c^{c-1}}[lambda] and F = M M^T {Q_c}[gamma],
 * vertex incidence lists (M^T's rows), and the crease matrix C as a per-edge sigma.  */
typedef struct {
    int32_t V, F, S, E, B;
    int32_t *slot_face;   /* [S] face of slot */
    int32_t *slot_next;   /* [S] next slot in the same face (Q_c) */
    int32_t *slot_prev;   /* [S] previous slot (Q_c^{c-1}) */
    int32_t *slot_edge;   /* [S] id of the edge v(slot) -> v(next slot) */
    int32_t *edge_lo, *edge_hi;      /* [E] */
    int32_t *edge_fwd, *edge_bwd;    /* [E] slot of lo->hi, slot of hi->lo, or -1 */
    int     *edge_bnd;    /* [E] 1 = E value 1 (boundary) */
    float   *edge_sigma;  /* [E] 0, crease sigma, or +inf for boundary (reading R6) */
    int     *edge_user_crease; /* [E] 1 = interior edge carrying a user crease (sigma > 0) */
    int32_t *ve_off, *ve_edge;   /* vertex -> incident edges, edge ids ascending */
    int32_t *vs_off, *vs_slot;   /* vertex -> incident slots (faces), slots ascending */
} topo;

static void topo_free(topo *T) {
    free(T->slot_face); free(T->slot_next); free(T->slot_prev); free(T->slot_edge);
    free(T->edge_lo); free(T->edge_hi); free(T->edge_fwd); free(T->edge_bwd); free(T->edge_bnd);
    free(T->edge_sigma); free(T->edge_user_crease);
    free(T->ve_off); free(T->ve_edge); free(T->vs_off); free(T->vs_slot);
    memset(T, 0, sizeof(*T));
}

typedef struct { int64_t key; int32_t slot; } keyslot;

static int cmp_keyslot(const void *pa, const void *pb) {
    const keyslot *a = (const keyslot *)pa, *b = (const keyslot *)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->slot > b->slot) - (a->slot < b->slot);
}

/* undirected key of an edge: (max, min) compared lexicographically (reading R1) */
static int64_t edge_key(int32_t a, int32_t b) {
    int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    return ((int64_t)hi << 32) | (int64_t)(uint32_t)lo;
}

static int find_edge(const topo *T, int32_t a, int32_t b) {
    int64_t key = edge_key(a, b);
    int32_t l = 0, h = T->E - 1;
    while (l <= h) {
        int32_t m = l + (h - l) / 2;
        int64_t k = edge_key(T->edge_lo[m], T->edge_hi[m]);
        if (k == key) return m;
        if (k < key) l = m + 1; else h = m - 1;
    }
    return -1;
}

/* slot of the reverse directed edge of slot s (F(j,i) of F(i,j)), or -1 */
static int32_t twin_slot(const topo *T, int32_t s) {
    int32_t e = T->slot_edge[s];
    return T->edge_fwd[e] == s ? T->edge_bwd[e] : T->edge_fwd[e];
}

static int build_topo(const om_mesh *in, topo *T, char *err, int errlen) {
    memset(T, 0, sizeof(*T));
    if (in->V < 0 || in->F < 0 || in->K < 0) { set_err(err, errlen, "negative count"); return OM_E_ARG; }
    if (in->F > 0 && (!in->face_off || !in->face_vtx)) { set_err(err, errlen, "null face arrays"); return OM_E_ARG; }
    if (in->V > 0 && !in->pos) { set_err(err, errlen, "null positions"); return OM_E_ARG; }
    if (in->K > 0 && (!in->crease || !in->sigma)) { set_err(err, errlen, "null crease arrays"); return OM_E_ARG; }
    const int32_t V = in->V, F = in->F;
    if (F > 0 && in->face_off[0] != 0) { set_err(err, errlen, "face_off[0] != 0"); return OM_E_MESH; }
    /* 1. face orders c_r = (M^T 1)_r (Eq. fo); validation (SURVEY.md §8(b) ALSUB_E_MESH) */
    for (int32_t r = 0; r < F; ++r) {
        int32_t c = in->face_off[r + 1] - in->face_off[r];
        if (c < 3) { set_err(err, errlen, "face %d has order %d < 3", r, c); return OM_E_MESH; }
        for (int32_t t = 0; t < c; ++t) {
            int32_t v = in->face_vtx[in->face_off[r] + t];
            if (v < 0 || v >= V) { set_err(err, errlen, "face %d: vertex index %d out of range", r, v); return OM_E_MESH; }
            for (int32_t u = 0; u < t; ++u)
                if (in->face_vtx[in->face_off[r] + u] == v) {
                    set_err(err, errlen, "face %d repeats vertex %d", r, v); return OM_E_MESH;
                }
        }
    }
    const int32_t S = F > 0 ? in->face_off[F] : 0;
    T->V = V; T->F = F; T->S = S;
    T->slot_face = xcalloc(S, 4); T->slot_next = xcalloc(S, 4); T->slot_prev = xcalloc(S, 4);
    T->slot_edge = xcalloc(S, 4);
    for (int32_t r = 0; r < F; ++r) {
        int32_t o = in->face_off[r], c = in->face_off[r + 1] - o;
        for (int32_t t = 0; t < c; ++t) {
            T->slot_face[o + t] = r;
            T->slot_next[o + t] = o + (t + 1) % c;       /* Q_c     */
            T->slot_prev[o + t] = o + (t + c - 1) % c;   /* Q_c^c-1 */
        }
    }
    /* 2. undirected edges: sort every slot's key (hi, lo); id = rank of the unique keys (R1) */
    keyslot *ks = xcalloc(S, sizeof(keyslot));
    for (int32_t s = 0; s < S; ++s) {
        ks[s].key = edge_key(in->face_vtx[s], in->face_vtx[T->slot_next[s]]);
        ks[s].slot = s;
    }
    qsort(ks, (size_t)S, sizeof(keyslot), cmp_keyslot);
    int32_t E = 0;
    for (int32_t i = 0; i < S; ++i)
        if (i == 0 || ks[i].key != ks[i - 1].key) ++E;
    T->E = E;
    T->edge_lo = xcalloc(E, 4); T->edge_hi = xcalloc(E, 4);
    T->edge_fwd = xcalloc(E, 4); T->edge_bwd = xcalloc(E, 4); T->edge_bnd = xcalloc(E, sizeof(int));
    T->edge_sigma = xcalloc(E, sizeof(float)); T->edge_user_crease = xcalloc(E, sizeof(int));
    int32_t e = -1;
    for (int32_t i = 0; i < S; ++i) {
        if (i == 0 || ks[i].key != ks[i - 1].key) {
            ++e;
            T->edge_hi[e] = (int32_t)(ks[i].key >> 32);
            T->edge_lo[e] = (int32_t)(ks[i].key & 0xffffffff);
            T->edge_fwd[e] = -1; T->edge_bwd[e] = -1;
        }
        int32_t s = ks[i].slot;
        T->slot_edge[s] = e;
        int32_t a = in->face_vtx[s];
        /* multiplicity of E(i,j) in {1,2}; a directed edge seen twice = orientation/non-manifold */
        if (a == T->edge_lo[e]) {
            if (T->edge_fwd[e] >= 0) { free(ks); set_err(err, errlen, "directed edge %d->%d appears twice", a, T->edge_hi[e]); return OM_E_NONMANIFOLD; }
            T->edge_fwd[e] = s;
        } else {
            if (T->edge_bwd[e] >= 0) { free(ks); set_err(err, errlen, "directed edge %d->%d appears twice", a, T->edge_lo[e]); return OM_E_NONMANIFOLD; }
            T->edge_bwd[e] = s;
        }
    }
    free(ks);
    int32_t B = 0;
    for (e = 0; e < E; ++e) {
        T->edge_bnd[e] = (T->edge_fwd[e] < 0 || T->edge_bwd[e] < 0);
        B += T->edge_bnd[e];
    }
    T->B = B;
    /* 3. vertex incidence: edges and slots per vertex (ascending ids) */
    T->ve_off = xcalloc((size_t)V + 1, 4); T->vs_off = xcalloc((size_t)V + 1, 4);
    for (e = 0; e < E; ++e) { T->ve_off[T->edge_lo[e] + 1]++; T->ve_off[T->edge_hi[e] + 1]++; }
    for (int32_t s = 0; s < S; ++s) T->vs_off[in->face_vtx[s] + 1]++;
    for (int32_t v = 0; v < V; ++v) { T->ve_off[v + 1] += T->ve_off[v]; T->vs_off[v + 1] += T->vs_off[v]; }
    T->ve_edge = xcalloc((size_t)2 * E, 4); T->vs_slot = xcalloc(S, 4);
    int32_t *fill = xcalloc((size_t)V + 1, 4);
    for (e = 0; e < E; ++e) {
        T->ve_edge[T->ve_off[T->edge_lo[e]] + fill[T->edge_lo[e]]++] = e;
        T->ve_edge[T->ve_off[T->edge_hi[e]] + fill[T->edge_hi[e]]++] = e;
    }
    memset(fill, 0, ((size_t)V + 1) * 4);
    for (int32_t s = 0; s < S; ++s) T->vs_slot[T->vs_off[in->face_vtx[s]] + fill[in->face_vtx[s]]++] = s;
    free(fill);
    /* 3b. fans around each vertex (reading R18).  Rotating slot h of v to twin(prev(h)) -- the
     * slot of v in the face across the edge entering v -- walks one fan.  A fan is open when it
     * starts at a slot whose outgoing edge is a boundary edge (twin(h) = -1).  Open fans are
     * allowed (a bowtie vertex; it ends up as a corner).  A closed fan together with any other
     * fan at the same vertex is non-manifold.                                                 */
    for (int32_t v = 0; v < V; ++v) {
        int32_t deg = T->vs_off[v + 1] - T->vs_off[v];
        if (deg == 0) continue;
        int32_t starts = 0, covered = 0;
        for (int32_t i = T->vs_off[v]; i < T->vs_off[v + 1]; ++i) {
            int32_t h = T->vs_slot[i];
            if (twin_slot(T, h) >= 0) continue;
            ++starts;
            int32_t n = 1;
            for (int32_t g = h; twin_slot(T, T->slot_prev[g]) >= 0 && n <= deg; ++n)
                g = twin_slot(T, T->slot_prev[g]);
            covered += n;
        }
        if (starts == 0) {   /* only closed fans: the one through the first slot must hold them all */
            int32_t h0 = T->vs_slot[T->vs_off[v]], g = h0, n = 0;
            do { g = twin_slot(T, T->slot_prev[g]); ++n; } while (g != h0 && n <= deg);
            covered = n;
        }
        if (covered != deg) {
            set_err(err, errlen, "vertex %d: its %d faces form a closed fan plus another fan", v, deg);
            return OM_E_NONMANIFOLD;
        }
    }
    /* 4. crease matrix C: sigma per edge; boundary edges are infinitely sharp (reading R6) */
    for (int32_t k = 0; k < in->K; ++k) {
        int32_t a = in->crease[2 * k], b = in->crease[2 * k + 1];
        float sg = in->sigma[k];
        if (a < 0 || a >= V || b < 0 || b >= V || a == b) { set_err(err, errlen, "crease %d: bad vertex pair (%d,%d)", k, a, b); return OM_E_CREASE; }
        if (isnan(sg) || sg < 0.0f) { set_err(err, errlen, "crease %d: sharpness %g", k, (double)sg); return OM_E_CREASE; }
        int32_t ce = find_edge(T, a, b);
        if (ce < 0) { set_err(err, errlen, "crease %d: (%d,%d) is not an edge", k, a, b); return OM_E_CREASE; }
        if (T->edge_user_crease[ce] < 0 || T->edge_sigma[ce] != 0.0f) { set_err(err, errlen, "crease %d: duplicate pair (%d,%d)", k, a, b); return OM_E_CREASE; }
        if (sg == 0.0f) { T->edge_user_crease[ce] = -1; continue; } /* zeros are elided from C; mark seen */
        T->edge_sigma[ce] = sg;
        T->edge_user_crease[ce] = 1;
    }
    for (e = 0; e < E; ++e) {
        if (T->edge_user_crease[e] < 0) T->edge_user_crease[e] = 0;
        if (T->edge_bnd[e]) { T->edge_sigma[e] = INFINITY; T->edge_user_crease[e] = 0; }
    }
    return OM_OK;
}

static void export_edges(const topo *T, om_edges *out) {
    out->E = T->E; out->B = T->B;
    out->edge_vtx = xcalloc((size_t)2 * T->E, 4);
    out->edge_face = xcalloc((size_t)2 * T->E, 4);
    for (int32_t e = 0; e < T->E; ++e) {
        out->edge_vtx[2 * e] = T->edge_lo[e];
        out->edge_vtx[2 * e + 1] = T->edge_hi[e];
        out->edge_face[2 * e] = T->edge_fwd[e] >= 0 ? T->slot_face[T->edge_fwd[e]] : -1;
        out->edge_face[2 * e + 1] = T->edge_bwd[e] >= 0 ? T->slot_face[T->edge_bwd[e]] : -1;
    }
}

int om_edges_of(const om_mesh *in, om_edges *edges, char *err, int errlen) {
    topo T;
    memset(edges, 0, sizeof(*edges));
    int st = build_topo(in, &T, err, errlen);
    if (st == OM_OK) export_edges(&T, edges);
    topo_free(&T);
    return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Crease quantities per vertex (Eqs. CC_crease_valency / CC_crease_vsharpness):
 * k_i = number of incident edges with sigma > 0 (boundary included, reading R6),
 * s_i = mean of their sigma (+inf if any is +inf, reading R9).                               */
static void crease_k_s(const topo *T, int32_t v, int *k, float *s, int32_t nb[2]) {
    int kk = 0, inf = 0;
    float sum = 0.0f;
    nb[0] = nb[1] = -1;
    for (int32_t i = T->ve_off[v]; i < T->ve_off[v + 1]; ++i) {
        int32_t e = T->ve_edge[i];
        float sg = T->edge_sigma[e];
        if (!(sg > 0.0f)) continue;
        if (kk < 2) nb[kk] = T->edge_lo[e] == v ? T->edge_hi[e] : T->edge_lo[e];
        ++kk;
        if (isinf(sg)) inf = 1; else sum += sg;
    }
    *k = kk;
    *s = kk == 0 ? 0.0f : (inf ? INFINITY : sum / (float)kk);
}

/* DeRose-style vertex rule on top of the scheme's smooth point (reading R7):
 *   k <= 1 : smooth;   k == 2 : crease 3/4 p + 1/8 (p_a + p_b);   k >= 3 : corner p;
 *   k >= 2 and s < 1 : (1 - s) smooth + s sharp.                                             */
static void vertex_rule(const topo *T, const double *P, int32_t v, const double smooth[3], double out[3]) {
    int k; float s; int32_t nb[2];
    crease_k_s(T, v, &k, &s, nb);
    if (k <= 1) { memcpy(out, smooth, sizeof(double) * 3); return; }
    double sharp[3];
    for (int d = 0; d < 3; ++d) {
        if (k == 2) sharp[d] = 0.75 * P[3 * v + d] + 0.125 * (P[3 * nb[0] + d] + P[3 * nb[1] + d]);
        else        sharp[d] = P[3 * v + d];
    }
    if (s >= 1.0f) { memcpy(out, sharp, sizeof(double) * 3); return; }
    double w = (double)s;
    for (int d = 0; d < 3; ++d) out[d] = (1.0 - w) * smooth[d] + w * sharp[d];
}

/* Edge rule on top of the scheme's smooth edge point (reading R7):
 *   sigma = 0: smooth;  sigma >= 1: midpoint;  0 < sigma < 1: (1 - sigma) smooth + sigma mid.  */
static void edge_rule(const topo *T, const double *P, int32_t e, const double smooth[3], double out[3]) {
    float sg = T->edge_sigma[e];
    int32_t a = T->edge_lo[e], b = T->edge_hi[e];
    if (!(sg > 0.0f)) { memcpy(out, smooth, sizeof(double) * 3); return; }
    double mid[3];
    for (int d = 0; d < 3; ++d) mid[d] = 0.5 * (P[3 * a + d] + P[3 * b + d]);
    if (sg >= 1.0f) { memcpy(out, mid, sizeof(double) * 3); return; }
    double w = (double)sg;
    for (int d = 0; d < 3; ++d) out[d] = (1.0 - w) * smooth[d] + w * mid[d];
}

/* Crease inheritance, P:L429-445 (variant of Chaikin, Eqs. sigma_ij / sigma_jk) with reading R8:
 * for each finite crease edge e = (a, b) and endpoint x, sigma_bar_x = mean sigma of the OTHER
 * finite sigma > 0 non-boundary crease edges at x (sigma_e itself if there are none);
 * child (x, ep_e) gets max(1/4 (sigma_bar_x + 3 sigma_e) - 1, 0); inf children stay inf;
 * zeros are dropped.  Children are emitted in ascending (ep, x) = child edge id order.      */
static int inherit_creases(const topo *T, int32_t ep_base, om_mesh *out) {
    int32_t cnt = 0;
    for (int32_t e = 0; e < T->E; ++e) if (T->edge_user_crease[e]) cnt += 2;
    out->crease = xcalloc((size_t)2 * cnt, 4);
    out->sigma = xcalloc(cnt, sizeof(float));
    int32_t K = 0;
    for (int32_t e = 0; e < T->E; ++e) {
        if (!T->edge_user_crease[e]) continue;
        float se = T->edge_sigma[e];
        int32_t ends[2] = {T->edge_lo[e], T->edge_hi[e]};
        for (int j = 0; j < 2; ++j) {
            int32_t x = ends[j];
            float child;
            if (isinf(se)) {
                child = INFINITY;
            } else {
                float sum = 0.0f;
                int n = 0;
                for (int32_t i = T->ve_off[x]; i < T->ve_off[x + 1]; ++i) {
                    int32_t o = T->ve_edge[i];
                    if (o == e || !T->edge_user_crease[o] || isinf(T->edge_sigma[o])) continue;
                    sum += T->edge_sigma[o];
                    ++n;
                }
                float sbar = n > 0 ? sum / (float)n : se;
                child = 0.25f * (sbar + 3.0f * se) - 1.0f;
                if (child < 0.0f) child = 0.0f;
            }
            if (child > 0.0f) {
                out->crease[2 * K] = x;
                out->crease[2 * K + 1] = ep_base + e;
                out->sigma[K] = child;
                ++K;
            }
        }
    }
    out->K = K;
    return OM_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Catmull-Clark (P:L178-220 classical rules; P:L222-368 ids; readings R1-R9).                 */
static int level_cc(const om_mesh *in, const topo *T, om_mesh *out, char *err, int errlen) {
    const int32_t V = T->V, F = T->F, E = T->E, S = T->S;
    const double *P = in->pos;
    int64_t Vn = (int64_t)V + F + E, Fn = S;
    if (Vn > INT32_MAX || (int64_t)4 * Fn > INT32_MAX) { set_err(err, errlen, "refined counts overflow int32"); return OM_E_OVERFLOW; }
    out->V = (int32_t)Vn; out->F = (int32_t)Fn;
    out->pos = xcalloc((size_t)3 * Vn, sizeof(double));
    double *fp = out->pos + 3 * (size_t)V;                 /* face points  at V + r      */
    double *epnt = out->pos + 3 * ((size_t)V + F);         /* edge points  at V + F + e  */
    /* face points f_r = (1/c_r) sum of the face's vertices (Eq. spla_fp) */
    OM_PARALLEL_FOR
    for (int32_t r = 0; r < F; ++r) {
        int32_t o = in->face_off[r], c = in->face_off[r + 1] - o;
        double acc[3] = {0, 0, 0};
        for (int32_t t = 0; t < c; ++t)
            for (int d = 0; d < 3; ++d) acc[d] += P[3 * in->face_vtx[o + t] + d];
        for (int d = 0; d < 3; ++d) fp[3 * r + d] = acc[d] / (double)c;
    }
    /* edge points e = 1/4 (p_k + p_l + f_r + f_s); boundary/crease rule */
    OM_PARALLEL_FOR
    for (int32_t e = 0; e < E; ++e) {
        int32_t a = T->edge_lo[e], b = T->edge_hi[e];
        double smooth[3];
        if (T->edge_bnd[e]) {
            for (int d = 0; d < 3; ++d) smooth[d] = 0.5 * (P[3 * a + d] + P[3 * b + d]);
        } else {
            int32_t r = T->slot_face[T->edge_fwd[e]], s = T->slot_face[T->edge_bwd[e]];
            for (int d = 0; d < 3; ++d)
                smooth[d] = 0.25 * (P[3 * a + d] + P[3 * b + d] + fp[3 * r + d] + fp[3 * s + d]);
        }
        edge_rule(T, P, e, smooth, epnt + 3 * (size_t)e);
    }
    /* vertex points S(p) = (1 - 2/n) p + 1/n^2 sum p_j + 1/n^2 sum f_j (Eq. pos_update, P:L202-209,
     * split P:L332-357); n = number of incident faces (Eq. vo; reading R4).       */
    OM_PARALLEL_FOR
    for (int32_t v = 0; v < V; ++v) {
        int32_t n = T->vs_off[v + 1] - T->vs_off[v];
        double smooth[3];
        if (n == 0) {  /* isolated vertex passes through (reading R17) */
            for (int d = 0; d < 3; ++d) smooth[d] = P[3 * v + d];
        } else {
            double sp[3] = {0, 0, 0}, sf[3] = {0, 0, 0};
            for (int32_t i = T->ve_off[v]; i < T->ve_off[v + 1]; ++i) {
                int32_t e = T->ve_edge[i];
                int32_t j = T->edge_lo[e] == v ? T->edge_hi[e] : T->edge_lo[e];
                for (int d = 0; d < 3; ++d) sp[d] += P[3 * j + d];
            }
            for (int32_t i = T->vs_off[v]; i < T->vs_off[v + 1]; ++i) {
                int32_t r = T->slot_face[T->vs_slot[i]];
                for (int d = 0; d < 3; ++d) sf[d] += fp[3 * r + d];
            }
            double nn = (double)n;
            for (int d = 0; d < 3; ++d)
                smooth[d] = (1.0 - 2.0 / nn) * P[3 * v + d] + sp[d] / (nn * nn) + sf[d] / (nn * nn);
        }
        vertex_rule(T, P, v, smooth, out->pos + 3 * (size_t)v);
    }
    /* topology: column r -> c_r quads (v_t, ep(v_t,v_t+1), fp_r, ep(v_t-1,v_t)) (R2) */
    out->face_off = xcalloc((size_t)Fn + 1, 4);
    out->face_vtx = xcalloc((size_t)4 * Fn, 4);
    OM_PARALLEL_FOR
    for (int32_t r = 0; r < F; ++r) {
        int32_t o = in->face_off[r], c = in->face_off[r + 1] - o;
        for (int32_t t = 0; t < c; ++t) {
            int32_t s = o + t, q = o + t;   /* child face index = off_r + t */
            int32_t *f = out->face_vtx + 4 * (size_t)q;
            f[0] = in->face_vtx[s];
            f[1] = V + F + T->slot_edge[s];
            f[2] = V + r;
            f[3] = V + F + T->slot_edge[T->slot_prev[s]];
        }
    }
    for (int64_t q = 0; q <= Fn; ++q) out->face_off[q] = (int32_t)(4 * q);
    return inherit_creases(T, V + F, out);
}

/* ------------------------------------------------------------------------------------------ */
/* Loop (Appendix B; readings R11, R12, R14).                                   */
static int level_loop(const om_mesh *in, const topo *T, om_mesh *out, char *err, int errlen) {
    const int32_t V = T->V, F = T->F, E = T->E;
    const double *P = in->pos;
    for (int32_t r = 0; r < F; ++r)
        if (in->face_off[r + 1] - in->face_off[r] != 3) { set_err(err, errlen, "Loop needs triangles (face %d)", r); return OM_E_SCHEME; }
    int64_t Vn = (int64_t)V + E, Fn = (int64_t)4 * F;
    if (Vn > INT32_MAX || 3 * Fn > INT32_MAX) { set_err(err, errlen, "refined counts overflow int32"); return OM_E_OVERFLOW; }
    out->V = (int32_t)Vn; out->F = (int32_t)Fn;
    out->pos = xcalloc((size_t)3 * Vn, sizeof(double));
    double *epnt = out->pos + 3 * (size_t)V;
    /* edge points: 3/8 (p_a + p_b) + 1/8 (p_G(a,b) + p_G(b,a)); G = vertex opposite the directed
     * edge (Eq. G); weights from Fig. loop_scheme (reading R11).  */
    OM_PARALLEL_FOR
    for (int32_t e = 0; e < E; ++e) {
        int32_t a = T->edge_lo[e], b = T->edge_hi[e];
        double smooth[3];
        if (T->edge_bnd[e]) {
            for (int d = 0; d < 3; ++d) smooth[d] = 0.5 * (P[3 * a + d] + P[3 * b + d]);
        } else {
            int32_t g1 = in->face_vtx[T->slot_prev[T->edge_fwd[e]]];
            int32_t g2 = in->face_vtx[T->slot_prev[T->edge_bwd[e]]];
            for (int d = 0; d < 3; ++d)
                smooth[d] = 0.375 * (P[3 * a + d] + P[3 * b + d]) + 0.125 * (P[3 * g1 + d] + P[3 * g2 + d]);
        }
        edge_rule(T, P, e, smooth, epnt + 3 * (size_t)e);
    }
    /* vertex update S(p) = (1 - n beta) p + beta sum p_j (Eq. loop_smooth) */
    OM_PARALLEL_FOR
    for (int32_t v = 0; v < V; ++v) {
        int32_t n = T->ve_off[v + 1] - T->ve_off[v];
        double smooth[3];
        if (n == 0) {
            for (int d = 0; d < 3; ++d) smooth[d] = P[3 * v + d];
        } else {
            double beta = om_loop_beta(n), sp[3] = {0, 0, 0};
            for (int32_t i = T->ve_off[v]; i < T->ve_off[v + 1]; ++i) {
                int32_t e = T->ve_edge[i];
                int32_t j = T->edge_lo[e] == v ? T->edge_hi[e] : T->edge_lo[e];
                for (int d = 0; d < 3; ++d) sp[d] += P[3 * j + d];
            }
            for (int d = 0; d < 3; ++d) smooth[d] = (1.0 - n * beta) * P[3 * v + d] + beta * sp[d];
        }
        vertex_rule(T, P, v, smooth, out->pos + 3 * (size_t)v);
    }
    /* topology: (k, e_kl, e_mk), (l, e_lm, e_kl), (m, e_mk, e_lm), (e_kl, e_lm, e_mk) */
    out->face_off = xcalloc((size_t)Fn + 1, 4);
    out->face_vtx = xcalloc((size_t)3 * Fn, 4);
    OM_PARALLEL_FOR
    for (int32_t r = 0; r < F; ++r) {
        int32_t o = in->face_off[r];
        int32_t ep[3];
        for (int t = 0; t < 3; ++t) ep[t] = V + T->slot_edge[o + t];   /* e_kl, e_lm, e_mk */
        for (int t = 0; t < 3; ++t) {
            int32_t *f = out->face_vtx + 3 * ((size_t)4 * r + t);
            f[0] = in->face_vtx[o + t];
            f[1] = ep[t];
            f[2] = ep[(t + 2) % 3];
        }
        int32_t *f = out->face_vtx + 3 * ((size_t)4 * r + 3);
        f[0] = ep[0]; f[1] = ep[1]; f[2] = ep[2];
    }
    for (int64_t q = 0; q <= Fn; ++q) out->face_off[q] = (int32_t)(3 * q);
    return inherit_creases(T, V, out);
}

/* ------------------------------------------------------------------------------------------ */
/* sqrt3 (Appendix A; readings R13, R14).                                         */
static int level_sqrt3(const om_mesh *in, const topo *T, om_mesh *out, char *err, int errlen) {
    const int32_t V = T->V, F = T->F;
    const double *P = in->pos;
    for (int32_t r = 0; r < F; ++r)
        if (in->face_off[r + 1] - in->face_off[r] != 3) { set_err(err, errlen, "sqrt3 needs triangles (face %d)", r); return OM_E_SCHEME; }
    if (T->B > 0) { set_err(err, errlen, "sqrt3 boundary rules are omitted by the paper (P:L1002)"); return OM_E_SCHEME; }
    for (int32_t e = 0; e < T->E; ++e)
        if (T->edge_user_crease[e]) { set_err(err, errlen, "sqrt3 has no crease rules"); return OM_E_SCHEME; }
    int64_t Vn = (int64_t)V + F, Fn = (int64_t)3 * F;
    if (Vn > INT32_MAX || 3 * Fn > INT32_MAX) { set_err(err, errlen, "refined counts overflow int32"); return OM_E_OVERFLOW; }
    out->V = (int32_t)Vn; out->F = (int32_t)Fn;
    out->pos = xcalloc((size_t)3 * Vn, sizeof(double));
    /* new vertex points: barycenters f = M^T P with (1,2,3) -> 1/3 */
    OM_PARALLEL_FOR
    for (int32_t r = 0; r < F; ++r) {
        int32_t o = in->face_off[r];
        for (int d = 0; d < 3; ++d)
            out->pos[3 * ((size_t)V + r) + d] =
                (P[3 * in->face_vtx[o] + d] + P[3 * in->face_vtx[o + 1] + d] + P[3 * in->face_vtx[o + 2] + d]) / 3.0;
    }
    /* S(p) = (1 - alpha) p + alpha/n sum p_j (Eqs. sqrt2, alpha) */
    OM_PARALLEL_FOR
    for (int32_t v = 0; v < V; ++v) {
        int32_t n = T->ve_off[v + 1] - T->ve_off[v];
        if (n == 0) { for (int d = 0; d < 3; ++d) out->pos[3 * (size_t)v + d] = P[3 * v + d]; continue; }
        double alpha = om_sqrt3_alpha(n), sp[3] = {0, 0, 0};
        for (int32_t i = T->ve_off[v]; i < T->ve_off[v + 1]; ++i) {
            int32_t e = T->ve_edge[i];
            int32_t j = T->edge_lo[e] == v ? T->edge_hi[e] : T->edge_lo[e];
            for (int d = 0; d < 3; ++d) sp[d] += P[3 * j + d];
        }
        for (int d = 0; d < 3; ++d) out->pos[3 * (size_t)v + d] = (1.0 - alpha) * P[3 * v + d] + alpha / n * sp[d];
    }
    /* topology: vertex p_k of triangle i = (p_k, p_l, p_m) contributes (p_k, fp_F(l,k), fp_i)
     * (CCW order, reading R13)                                                  */
    out->face_off = xcalloc((size_t)Fn + 1, 4);
    out->face_vtx = xcalloc((size_t)3 * Fn, 4);
    OM_PARALLEL_FOR
    for (int32_t r = 0; r < F; ++r) {
        int32_t o = in->face_off[r];
        for (int t = 0; t < 3; ++t) {
            int32_t s = o + t, e = T->slot_edge[s];
            int32_t rev = (T->edge_fwd[e] == s) ? T->edge_bwd[e] : T->edge_fwd[e];   /* slot l -> k */
            int32_t *f = out->face_vtx + 3 * ((size_t)3 * r + t);
            f[0] = in->face_vtx[s];
            f[1] = V + T->slot_face[rev];
            f[2] = V + r;
        }
    }
    for (int64_t q = 0; q <= Fn; ++q) out->face_off[q] = (int32_t)(3 * q);
    out->K = 0; out->crease = xcalloc(0, 4); out->sigma = xcalloc(0, 4);
    return OM_OK;
}

int om_level(int scheme, const om_mesh *in, om_mesh *out, om_edges *edges, char *err, int errlen) {
    memset(out, 0, sizeof(*out));
    if (edges) memset(edges, 0, sizeof(*edges));
    if (!in || scheme < OM_CC || scheme > OM_SQRT3) { set_err(err, errlen, "bad argument"); return OM_E_ARG; }
    topo T;
    int st = build_topo(in, &T, err, errlen);
    if (st == OM_OK) {
        if (scheme == OM_CC) st = level_cc(in, &T, out, err, errlen);
        else if (scheme == OM_LOOP) st = level_loop(in, &T, out, err, errlen);
        else st = level_sqrt3(in, &T, out, err, errlen);
    }
    if (st == OM_OK && edges) export_edges(&T, edges);
    if (st != OM_OK) om_mesh_free(out);
    topo_free(&T);
    return st;
}
