// reorder.cpp -- reverse Cuthill-McKee ordering of the control mesh (
// PAPER.md "Mesh reordering": RCM on the graph Laplacian of the mesh, the rows of M
// permuted, the columns (faces) sorted by their first non-zero).
//
// An offline host preprocess, like the paper's precomputed reorderings: it runs once per
// control mesh, outside the refinement path, on a mesh of <= ~10^5 vertices.  Deterministic tie
// breaking (degree, then id) so that tests/ can check it index for index against oracle/rcm.py:
//   start vertex  George-Liu pseudo-peripheral node: min-degree vertex of the component, then
//                 repeatedly the min-degree vertex of the last BFS level while the eccentricity grows
//   CM order      BFS; each dequeued vertex appends its unvisited neighbours by (degree, id)
//   RCM           all components' CM orders concatenated and reversed
//   faces         by min new vertex id, ties in the original order (reading R24)
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "alsub.h"

namespace alsub {
alsub_status set_error(alsub_status st, const char *msg);
}

namespace {

struct Graph {
    std::vector<int32_t> off, adj;
    int32_t deg(int32_t v) const { return off[v + 1] - off[v]; }
};

// BFS level structure from r over the graph; returns the number of levels and the last level
int32_t bfs_levels(const Graph &g, int32_t r, std::vector<int32_t> &mark, int32_t stamp, std::vector<int32_t> &last) {
    std::vector<int32_t> cur{r}, nxt;
    mark[r] = stamp;
    int32_t nlev = 1;
    for (;;) {
        nxt.clear();
        for (int32_t v : cur)
            for (int32_t q = g.off[v]; q < g.off[v + 1]; ++q) {
                const int32_t w = g.adj[q];
                if (mark[w] != stamp) {
                    mark[w] = stamp;
                    nxt.push_back(w);
                }
            }
        if (nxt.empty()) break;
        cur.swap(nxt);
        ++nlev;
    }
    last = cur;
    return nlev;
}

}  // namespace

extern "C" alsub_status alsub_rcm_order(const int32_t *face_off, const int32_t *face_vtx, int32_t num_faces,
                                        int32_t num_verts, int32_t *perm_vtx, int32_t *perm_face) {
    if (num_faces < 0 || num_verts < 0 || (num_faces > 0 && (!face_off || !face_vtx)) ||
        (num_verts > 0 && !perm_vtx) || (num_faces > 0 && !perm_face))
        return alsub::set_error(ALSUB_E_ARG, "bad argument");
    const int32_t V = num_verts, F = num_faces;
    // vertex graph of the mesh edges (the off-diagonal pattern of the graph Laplacian): both
    // directions of every face side bucketed by vertex (counting sort), each list sorted and
    // de-duplicated -- O(slots), not a global sort of the pairs
    for (int32_t r = 0; r < F; ++r) {
        const int32_t o = face_off[r], c = face_off[r + 1] - o;
        if (c < 1) return alsub::set_error(ALSUB_E_MESH, "face with no vertices");
        for (int32_t t = 0; t < c; ++t) {
            const int32_t a = face_vtx[o + t];
            if (a < 0 || a >= V) return alsub::set_error(ALSUB_E_MESH, "vertex index out of range");
        }
    }
    std::vector<int32_t> cnt((size_t)V + 1, 0);
    for (int32_t r = 0; r < F; ++r) {
        const int32_t o = face_off[r], c = face_off[r + 1] - o;
        for (int32_t t = 0; t < c; ++t) {
            const int32_t a = face_vtx[o + t], b = face_vtx[o + (t + 1) % c];
            if (a == b) continue;
            ++cnt[a + 1];
            ++cnt[b + 1];
        }
    }
    for (int32_t v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
    std::vector<int32_t> raw((size_t)cnt[V]), cur(cnt.begin(), cnt.end() - 1);
    for (int32_t r = 0; r < F; ++r) {
        const int32_t o = face_off[r], c = face_off[r + 1] - o;
        for (int32_t t = 0; t < c; ++t) {
            const int32_t a = face_vtx[o + t], b = face_vtx[o + (t + 1) % c];
            if (a == b) continue;
            raw[cur[a]++] = b;
            raw[cur[b]++] = a;
        }
    }
    Graph g;
    g.off.assign((size_t)V + 1, 0);
    g.adj.reserve(raw.size());
    for (int32_t v = 0; v < V; ++v) {
        int32_t *lo = raw.data() + cnt[v], *hi = raw.data() + cnt[v + 1];
        std::sort(lo, hi);
        hi = std::unique(lo, hi);
        g.adj.insert(g.adj.end(), lo, hi);
        g.off[v + 1] = (int32_t)g.adj.size();
    }
    auto less_deg = [&](int32_t a, int32_t b) { return g.deg(a) != g.deg(b) ? g.deg(a) < g.deg(b) : a < b; };

    std::vector<int32_t> mark((size_t)V, -1), order, comp_last, last;
    std::vector<char> visited((size_t)V, 0);
    order.reserve((size_t)V);
    int32_t stamp = 0;
    for (int32_t s = 0; s < V; ++s) {
        if (visited[s]) continue;
        // the component of s and its minimum-degree vertex
        std::vector<int32_t> comp{s};
        {
            const int32_t st = stamp++;
            mark[s] = st;
            for (size_t i = 0; i < comp.size(); ++i)
                for (int32_t q = g.off[comp[i]]; q < g.off[comp[i] + 1]; ++q)
                    if (mark[g.adj[q]] != st) {
                        mark[g.adj[q]] = st;
                        comp.push_back(g.adj[q]);
                    }
        }
        int32_t r = *std::min_element(comp.begin(), comp.end(), less_deg);
        int32_t ecc = bfs_levels(g, r, mark, stamp++, last);
        for (;;) {
            const int32_t x = *std::min_element(last.begin(), last.end(), less_deg);
            const int32_t ex = bfs_levels(g, x, mark, stamp++, comp_last);
            if (ex > ecc) {
                r = x;
                ecc = ex;
                last.swap(comp_last);
            } else {
                break;
            }
        }
        // Cuthill-McKee BFS from r
        size_t head = order.size();
        order.push_back(r);
        visited[r] = 1;
        std::vector<int32_t> nb;
        while (head < order.size()) {
            const int32_t v = order[head++];
            nb.clear();
            for (int32_t q = g.off[v]; q < g.off[v + 1]; ++q)
                if (!visited[g.adj[q]]) nb.push_back(g.adj[q]);
            std::sort(nb.begin(), nb.end(), less_deg);
            for (int32_t w : nb) {
                visited[w] = 1;
                order.push_back(w);
            }
        }
    }
    std::vector<int32_t> newid((size_t)V);
    for (int32_t i = 0; i < V; ++i) {
        perm_vtx[i] = order[(size_t)V - 1 - i];
        newid[perm_vtx[i]] = i;
    }
    // faces by their minimum new vertex id, ties in the original order: a stable counting sort
    std::vector<int32_t> key((size_t)F), start((size_t)V + 1, 0);
    for (int32_t r = 0; r < F; ++r) {
        int32_t k = INT32_MAX;
        for (int32_t h = face_off[r]; h < face_off[r + 1]; ++h) k = std::min(k, newid[face_vtx[h]]);
        key[r] = k;
        ++start[k + 1];
    }
    for (int32_t v = 0; v < V; ++v) start[v + 1] += start[v];
    for (int32_t r = 0; r < F; ++r) perm_face[start[key[r]]++] = r;
    return ALSUB_OK;
}
