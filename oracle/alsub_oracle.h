/*
 * alsub_oracle.h -- plain, slow, obviously-correct CPU oracle for ONE uniform refinement level
 * of AlSub (arXiv 1809.06047).  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path in paper_1809_06047_b200/.
 *
 * Precision: positions in fp64; crease sharpness in fp32 (reading R10).
 * Every rule cites the PAPER.md line (P:Lnnn) or DESIGN.md reading (Rnn) it follows.
 */
#ifndef ALSUB_ORACLE_H
#define ALSUB_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OM_CC = 0, OM_LOOP = 1, OM_SQRT3 = 2 };
enum { OM_OK = 0, OM_E_ARG = 1, OM_E_MESH = 2, OM_E_NONMANIFOLD = 3, OM_E_SCHEME = 4, OM_E_CREASE = 5,
       OM_E_OVERFLOW = 6, OM_E_NOMEM = 7 };

/* A polygon mesh = the mesh matrix M in CSC form: column r = face r,
 * rows = its vertices in cyclic (CCW) order.  Creases = the upper triangle of C. */
typedef struct {
    int32_t V, F;
    int32_t *face_off;   /* [F+1] */
    int32_t *face_vtx;   /* [face_off[F]] */
    double  *pos;        /* [3V] */
    int32_t K;
    int32_t *crease;     /* [2K] (lo, hi) pairs, lo < hi, ascending (hi, lo) */
    float   *sigma;      /* [K]  > 0, +inf allowed */
} om_mesh;

/* Edge tables of the level that was refined: E = M M^T with {Q_c + Q_c^{c-1}};
 * edge id = rank of (hi, lo) in ascending order (reading R1); F(i,j). */
typedef struct {
    int32_t E, B;
    int32_t *edge_vtx;   /* [2E] (lo, hi) */
    int32_t *edge_face;  /* [2E] face containing lo->hi, face containing hi->lo; -1 = none */
} om_edges;

/* Refine `in` by one level of `scheme`.  On OM_OK, *out holds the child mesh and *edges the
 * parent's edge tables (both malloc'd; free with om_mesh_free / om_edges_free).  On error the
 * outputs are left empty and err (if non-null) receives a message. */
int  om_level(int scheme, const om_mesh *in, om_mesh *out, om_edges *edges, char *err, int errlen);

/* Validate and enumerate the edges of a mesh without refining it (creases are looked up). */
int  om_edges_of(const om_mesh *in, om_edges *edges, char *err, int errlen);

void om_mesh_free(om_mesh *m);
void om_edges_free(om_edges *e);

/* Scheme weights, exposed for the pins (P:L1044-1046 beta, P:L990-992 alpha). */
double om_loop_beta(int n);
double om_sqrt3_alpha(int n);

/* Threads of the OpenMP build (liboracle_omp.so); returns the count in use (1 in the serial build). */
int om_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
