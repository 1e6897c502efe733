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
#include <numeric>
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
    // vertex graph of the mesh edges (the off-diagonal pattern of the graph Laplacian)
    std::vector<std::pair<int32_t, int32_t>> pairs;
    for (int32_t r = 0; r < F; ++r) {
        const int32_t o = face_off[r], c = face_off[r + 1] - o;
        if (c < 1) return alsub::set_error(ALSUB_E_MESH, "face with no vertices");
        for (int32_t t = 0; t < c; ++t) {
            const int32_t a = face_vtx[o + t], b = face_vtx[o + (t + 1) % c];
            if (a < 0 || a >= V || b < 0 || b >= V) return alsub::set_error(ALSUB_E_MESH, "vertex index out of range");
            if (a == b) continue;
            pairs.emplace_back(a, b);
            pairs.emplace_back(b, a);
        }
    }
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
    Graph g;
    g.off.assign((size_t)V + 1, 0);
    g.adj.resize(pairs.size());
    for (size_t i = 0; i < pairs.size(); ++i) {
        ++g.off[pairs[i].first + 1];
        g.adj[i] = pairs[i].second;
    }
    for (int32_t v = 0; v < V; ++v) g.off[v + 1] += g.off[v];
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
    std::vector<int32_t> key((size_t)F);
    for (int32_t r = 0; r < F; ++r) {
        int32_t k = INT32_MAX;
        for (int32_t h = face_off[r]; h < face_off[r + 1]; ++h) k = std::min(k, newid[face_vtx[h]]);
        key[r] = k;
    }
    std::vector<int32_t> fo((size_t)F);
    std::iota(fo.begin(), fo.end(), 0);
    std::stable_sort(fo.begin(), fo.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    std::copy(fo.begin(), fo.end(), perm_face);
    return ALSUB_OK;
}
