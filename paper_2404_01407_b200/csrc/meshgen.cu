// meshgen.cu -- device-side mesh preprocessing: the median-dual
// geometry of the structured hex / Kuhn-tet sector meshes the five configurations use.
//
// The host restatement is mesh.py::_sector_dual_host; the kernels evaluate the same
// expressions in the same order (no FMA contraction: --fmad=false), so the results are
// bitwise equal:
//   * per cell and template edge (12 hex edges, or 6 Kuhn tets x 6 edges) the dual-face
//     piece S = 0.5 (cen - m) x (c2 - c1), oriented along the edge (sign of S.(xq - xp))
//     and stored against the ascending node pair (lo, hi), at position template x ncell +
//     cell (the host's concatenation order);
//   * per edge the pieces summed from 0.0 in that order: a stable radix sort of the
//     edge keys lo * n + hi carries the positions, and one thread per unique edge adds its
//     run sequentially (the np.unique / np.bincount of the host);
//   * per node its volume, ((0 + B_0) + B_1) + ..., B_c = the volume share of the one cell
//     (or Kuhn tet) having the node as corner c.
// The reference has no 3D generator (its meshes are the quasi-1D nozzle's, mesh.cpp);
// what it shares with this code is downstream: the edge -> block CSR step (make_pattern,
// sparse.cpp:91-117: fnlh_make_pattern) and the node -> face adjacency
// (Mesh::build_adjacency, mesh.cpp:44-59: fnlh_mesh_derive, which also derives the face
// areas / unit normals / viscous weights and the slip-wall closure of mesh.py::from_faces).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include <memory>
#include <vector>

#include "capi_util.hpp"
#include "fnlh_b200.h"

namespace fnlh {
namespace {

constexpr int kT = 256;
inline int nb(long long n) { return static_cast<int>((n + kT - 1) / kT); }

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 operator/(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {  // mesh.py::_cross
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double dot3(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ double tet_vol(V3 a, V3 b, V3 c, V3 d) { return fabs(dot3(b - a, cross(c - a, d - a))) / 6.0; }

// template tables, built on the host with the same loops as mesh.py
struct Tables {
    int hex_p[12], hex_q[12], hex_f1[12][4], hex_f2[12][4];  // _HEX_EDGES, _hex_edge_faces
    int kuhn[6][4];                                          // _KUHN
    int pair_p[6], pair_q[6], pair_r[6], pair_s[6];          // combinations(range(4), 2) + the others
};

Tables make_tables() {
    Tables t{};
    int e = 0;
    for (int d = 0; d < 3; ++d)
        for (int p = 0; p < 8; ++p) {
            if ((p >> d) & 1) continue;
            const int q = p | (1 << d);
            t.hex_p[e] = p;
            t.hex_q[e] = q;
            int nf = 0;
            for (int ax = 0; ax < 3; ++ax) {
                if (ax == d) continue;
                const int bit = (p >> ax) & 1;
                int k = 0;
                for (int v = 0; v < 8; ++v)
                    if (((v >> ax) & 1) == bit) (nf == 0 ? t.hex_f1[e] : t.hex_f2[e])[k++] = v;
                ++nf;
            }
            ++e;
        }
    const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int k = 0; k < 6; ++k) {
        const int a = perm[k][0], b = perm[k][1];
        t.kuhn[k][0] = 0;
        t.kuhn[k][1] = 1 << a;
        t.kuhn[k][2] = (1 << a) | (1 << b);
        t.kuhn[k][3] = 7;
    }
    int c = 0;
    for (int p = 0; p < 4; ++p)
        for (int q = p + 1; q < 4; ++q) {
            t.pair_p[c] = p;
            t.pair_q[c] = q;
            int o[2], k = 0;
            for (int v = 0; v < 4; ++v)
                if (v != p && v != q) o[k++] = v;
            t.pair_r[c] = o[0];
            t.pair_s[c] = o[1];
            ++c;
        }
    return t;
}

struct Dims {
    int ci, cj, ck, nj, nju, nk, periodic;
    long long ncell, n;
};

__device__ __forceinline__ void cell_corners(const Dims& d, long long cell, const double* __restrict__ Xu, V3 (&P)[8],
                                             long long (&id)[8]) {
    const int kc = (int)(cell % d.ck);
    const int jc = (int)((cell / d.ck) % d.cj);
    const int ic = (int)(cell / ((long long)d.ck * d.cj));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int i = ic + (c & 1), j = jc + ((c >> 1) & 1), k = kc + ((c >> 2) & 1);
        const long long u = ((long long)i * d.nju + j) * d.nk + k;
        P[c] = {Xu[3 * u], Xu[3 * u + 1], Xu[3 * u + 2]};
        id[c] = ((long long)i * d.nj + (j % d.nj)) * d.nk + k;
    }
}

__device__ __forceinline__ void put_edge(const Dims& d, long long slot, long long p_id, long long q_id, V3 S, V3 xp,
                                         V3 xq, unsigned long long* __restrict__ keys, double* __restrict__ vecs) {
    const double g = dot3(S, xq - xp);
    const double sgn = g > 0.0 ? 1.0 : (g < 0.0 ? -1.0 : 0.0);  // np.sign
    S = {S.x * sgn, S.y * sgn, S.z * sgn};
    const long long lo = p_id < q_id ? p_id : q_id, hi = p_id < q_id ? q_id : p_id;
    const double flip = p_id < q_id ? 1.0 : -1.0;
    keys[slot] = (unsigned long long)(lo * d.n + hi);
    vecs[3 * slot] = S.x * flip;
    vecs[3 * slot + 1] = S.y * flip;
    vecs[3 * slot + 2] = S.z * flip;
}

__global__ void k_hex_cells(Dims d, Tables t, const double* __restrict__ Xu, unsigned long long* __restrict__ keys,
                            double* __restrict__ vecs, double* __restrict__ vcell) {
    const long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (cell >= d.ncell) return;
    V3 P[8];
    long long id[8];
    cell_corners(d, cell, Xu, P, id);
    V3 cen = P[0];
#pragma unroll
    for (int c = 1; c < 8; ++c) cen = cen + P[c];
    cen = cen / 8.0;
    for (int e = 0; e < 12; ++e) {
        const int p = t.hex_p[e], q = t.hex_q[e];
        const V3 m = 0.5 * (P[p] + P[q]);
        V3 c1 = P[t.hex_f1[e][0]], c2 = P[t.hex_f2[e][0]];
        for (int k = 1; k < 4; ++k) {
            c1 = c1 + P[t.hex_f1[e][k]];
            c2 = c2 + P[t.hex_f2[e][k]];
        }
        c1 = c1 / 4.0;
        c2 = c2 / 4.0;
        put_edge(d, e * d.ncell + cell, id[p], id[q], 0.5 * cross(cen - m, c2 - c1), P[p], P[q], keys, vecs);
    }
    double vc = 0.0;
    for (int k = 0; k < 6; ++k) vc = vc + tet_vol(P[t.kuhn[k][0]], P[t.kuhn[k][1]], P[t.kuhn[k][2]], P[t.kuhn[k][3]]);
    vcell[cell] = vc;
}

__global__ void k_tet_cells(Dims d, Tables t, const double* __restrict__ Xu, unsigned long long* __restrict__ keys,
                            double* __restrict__ vecs, double* __restrict__ vtet) {
    const long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (cell >= d.ncell) return;
    V3 P[8];
    long long id[8];
    cell_corners(d, cell, Xu, P, id);
    for (int k = 0; k < 6; ++k) {
        V3 T[4];
        long long tid[4];
        for (int c = 0; c < 4; ++c) {
            T[c] = P[t.kuhn[k][c]];
            tid[c] = id[t.kuhn[k][c]];
        }
        const V3 cen = (((T[0] + T[1]) + T[2]) + T[3]) / 4.0;
        vtet[k * d.ncell + cell] = tet_vol(T[0], T[1], T[2], T[3]);
        for (int e = 0; e < 6; ++e) {
            const int p = t.pair_p[e], q = t.pair_q[e], r = t.pair_r[e], s = t.pair_s[e];
            const V3 m = 0.5 * (T[p] + T[q]);
            const V3 c1 = ((T[p] + T[q]) + T[r]) / 3.0;
            const V3 c2 = ((T[p] + T[q]) + T[s]) / 3.0;
            put_edge(d, (k * 6 + e) * d.ncell + cell, tid[p], tid[q], 0.5 * cross(cen - m, c2 - c1), T[p], T[q], keys,
                     vecs);
        }
    }
}

// the cell having node (i, j, k) as corner c, or -1 (periodic pitch wraps j)
__device__ __forceinline__ long long corner_cell(const Dims& d, int i, int j, int k, int c) {
    const int ic = i - (c & 1), kc = k - ((c >> 2) & 1);
    int jc = j - ((c >> 1) & 1);
    if (d.periodic && jc < 0) jc += d.cj;
    if (ic < 0 || ic >= d.ci || jc < 0 || jc >= d.cj || kc < 0 || kc >= d.ck) return -1;
    return ((long long)ic * d.cj + jc) * d.ck + kc;
}

__global__ void k_node_vol(Dims d, Tables t, int tets, const double* __restrict__ vc, double* __restrict__ vol) {
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= d.n) return;
    const int k = (int)(v % d.nk), j = (int)((v / d.nk) % d.nj), i = (int)(v / ((long long)d.nk * d.nj));
    double acc = 0.0;
    if (!tets) {
        for (int c = 0; c < 8; ++c) {
            const long long cell = corner_cell(d, i, j, k, c);
            acc = acc + (cell >= 0 ? vc[cell] / 8.0 : 0.0);
        }
    } else {
        for (int q = 0; q < 6; ++q)
            for (int c = 0; c < 4; ++c) {
                const long long cell = corner_cell(d, i, j, k, t.kuhn[q][c]);
                acc = acc + (cell >= 0 ? vc[q * d.ncell + cell] / 4.0 : 0.0);
            }
    }
    vol[v] = acc;
}

__global__ void k_iota(long long m, long long* __restrict__ o) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < m) o[i] = i;
}

__global__ void k_heads(long long m, const unsigned long long* __restrict__ k, int* __restrict__ head) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < m) head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

__global__ void k_starts(long long m, const int* __restrict__ head, const long long* __restrict__ seg,
                         long long* __restrict__ start) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < m && head[i]) start[seg[i] - 1] = i;
}

// one thread per unique edge: its pieces summed from 0.0 in ascending position order
__global__ void k_edge_sums(long long nu, long long m, long long n, const long long* __restrict__ start,
                            const unsigned long long* __restrict__ k, const long long* __restrict__ pos,
                            const double* __restrict__ vecs, long long* __restrict__ ea, long long* __restrict__ eb,
                            double* __restrict__ en) {
    const long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (u >= nu) return;
    const long long s = start[u], e = u + 1 < nu ? start[u + 1] : m;
    double x = 0.0, y = 0.0, z = 0.0;
    for (long long q = s; q < e; ++q) {
        const long long p = pos[q];
        x = x + vecs[3 * p];
        y = y + vecs[3 * p + 1];
        z = z + vecs[3 * p + 2];
    }
    const long long key = (long long)k[s];
    ea[u] = key / n;
    eb[u] = key % n;
    en[3 * u] = x;
    en[3 * u + 1] = y;
    en[3 * u + 2] = z;
}

// ---- make_pattern (sparse.cpp:91-117) ---------------------------------------------
__global__ void k_pattern_keys(int rows, long long ne, const int* __restrict__ ea, const int* __restrict__ eb,
                               unsigned long long* __restrict__ keys, int* __restrict__ bad) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const unsigned long long R = (unsigned long long)rows;
    if (t < rows) keys[t] = (unsigned long long)t * R + (unsigned long long)t;
    if (t < ne) {
        const int a = ea[t], c = eb[t];
        if (a < 0 || a >= rows || c < 0 || c >= rows) {
            atomicExch(bad, 1);
            keys[rows + 2 * t] = keys[rows + 2 * t + 1] = 0ull;
            return;
        }
        keys[rows + 2 * t] = (unsigned long long)a * R + (unsigned long long)c;
        keys[rows + 2 * t + 1] = (unsigned long long)c * R + (unsigned long long)a;
    }
}

// unique sorted keys -> col_idx; row_ptr[r] = first entry of row r; diag_idx[r]
__global__ void k_pattern_fill(long long nnz, int rows, const unsigned long long* __restrict__ u,
                               int* __restrict__ row_ptr, int* __restrict__ col_idx, int* __restrict__ diag_idx) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const unsigned long long R = (unsigned long long)rows;
    const int r = (int)(u[e] / R), c = (int)(u[e] % R);
    col_idx[e] = c;
    if (r == c) diag_idx[r] = (int)e;
    if (e == 0 || (int)(u[e - 1] / R) != r) row_ptr[r] = (int)e;
    if (e == nnz - 1) row_ptr[rows] = (int)nnz;
}

// ---- Mesh::build_adjacency (mesh.cpp:44-59) and the derived face / node arrays -------
// events (node, face) in face order: fa then fb (interior faces); sign +1 / -1
__global__ void k_face_events(int nf, const int* __restrict__ fa, const int* __restrict__ fb,
                              unsigned int* __restrict__ node, int* __restrict__ ev) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    node[2 * f] = (unsigned int)fa[f];
    ev[2 * f] = 2 * f;
    node[2 * f + 1] = fb[f] >= 0 ? (unsigned int)fb[f] : 0xffffffffu;  // boundary: sorted past every node
    ev[2 * f + 1] = 2 * f + 1;
}

__global__ void k_node_ptr(long long m, int n, const unsigned int* __restrict__ node, int* __restrict__ nf_ptr) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= m) return;
    const unsigned int v = node[e];
    const unsigned int prev = e == 0 ? 0xffffffffu : node[e - 1];
    if (v != 0xffffffffu && (e == 0 || prev != v)) {
        // nodes without faces between prev and v get the same start
        const int lo = e == 0 ? 0 : (int)prev + 1;
        for (int q = lo; q <= (int)v; ++q) nf_ptr[q] = (int)e;
    }
    if (v != 0xffffffffu && (e == m - 1 || node[e + 1] != v)) {
        if (e == m - 1 || node[e + 1] == 0xffffffffu)
            for (int q = (int)v + 1; q <= n; ++q) nf_ptr[q] = (int)(e + 1);
    }
}

// per face: area, unit normal, viscous weight; per node: face list, closure, boundary flag
__global__ void k_face_derived(int nf, const double* __restrict__ fn, const int* __restrict__ fa,
                               const int* __restrict__ fb, const double* __restrict__ X, double* __restrict__ farea,
                               double* __restrict__ fnh, double* __restrict__ fvis) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const double x = fn[3 * f], y = fn[3 * f + 1], z = fn[3 * f + 2];
    const double a = sqrt((x * x + y * y) + z * z);
    farea[f] = a;
    fnh[3 * f] = x / a;
    fnh[3 * f + 1] = y / a;
    fnh[3 * f + 2] = z / a;
    double w = 0.0;
    if (X && fb[f] >= 0) {
        const long long p = fa[f], q = fb[f];
        const double dx = X[3 * q] - X[3 * p], dy = X[3 * q + 1] - X[3 * p + 1], dz = X[3 * q + 2] - X[3 * p + 2];
        w = a / sqrt((dx * dx + dy * dy) + dz * dz);
    }
    fvis[f] = w;
}

__global__ void k_node_derived(int n, const int* __restrict__ nf_ptr, const int* __restrict__ ev_s,
                               const double* __restrict__ fn, const int* __restrict__ fb, int* __restrict__ nf_idx,
                               double* __restrict__ closure, int* __restrict__ bflag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = 0.0, y = 0.0, z = 0.0;
    int bnd = 0;
    for (int q = nf_ptr[i]; q < nf_ptr[i + 1]; ++q) {
        const int e = ev_s[q], f = e >> 1;
        const double sg = (e & 1) ? -1.0 : 1.0;
        nf_idx[q] = f;
        x = x + fn[3 * f] * sg;
        y = y + fn[3 * f + 1] * sg;
        z = z + fn[3 * f + 2] * sg;
        if (fb[f] < 0) bnd = 1;
    }
    closure[3 * i] = x;
    closure[3 * i + 1] = y;
    closure[3 * i + 2] = z;
    bflag[i] = bnd;
}

int key_bits(long long n) {
    const unsigned long long top = (unsigned long long)n * (unsigned long long)n;
    int b = 1;
    while (b < 64 && (top >> b)) ++b;
    return b;
}

}  // namespace

struct SectorDual {
    long long n = 0, ne = 0;
    DeviceBuffer<long long> ea, eb;
    DeviceBuffer<double> en, vol;
};


// ---- Reverse Cuthill-McKee (scipy.sparse.csgraph.reverse_cuthill_mckee, the host
// ordering step of mesh.py::structured_sector) as a level-synchronous BFS.  Sequential
// Cuthill-McKee appends, for each dequeued node u in order, its unvisited neighbours by
// ascending degree (stable in CSR order); a node is taken by the first u that sees it.  So
// level L+1 is exactly its nodes sorted by (position of the claiming parent, degree, CSR
// slot in that parent), the claim being the minimum (parent position, slot): one
// atomicMin per (frontier node, neighbour), one radix sort per level.
__global__ void k_rcm_claim(int nf, const int* __restrict__ frontier, const long long* __restrict__ pos,
                            const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                            const int* __restrict__ visited, unsigned long long* __restrict__ claim,
                            int* __restrict__ mark, int* __restrict__ next, int* __restrict__ nnext) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nf) return;
    const int u = frontier[t];
    const unsigned long long pu = (unsigned long long)pos[u];
    for (int e = row_ptr[u], slot = 0; e < row_ptr[u + 1]; ++e, ++slot) {
        const int v = col_idx[e];
        if (visited[v]) continue;
        atomicMin(claim + v, (pu << 8) | (unsigned long long)slot);
        if (atomicExch(mark + v, 1) == 0) next[atomicAdd(nnext, 1)] = v;
    }
}
__global__ void k_rcm_keys(int nn, const int* __restrict__ next, const unsigned long long* __restrict__ claim,
                           const int* __restrict__ row_ptr, unsigned long long* __restrict__ keys) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nn) return;
    const int v = next[t];
    const unsigned long long c = claim[v];
    const unsigned long long deg = (unsigned long long)(row_ptr[v + 1] - row_ptr[v]);
    keys[t] = ((c >> 8) << 16) | (deg << 8) | (c & 255ull);
}
__global__ void k_rcm_assign(int nn, const int* __restrict__ sorted, long long base, long long* __restrict__ pos,
                             int* __restrict__ visited, int* __restrict__ order) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nn) return;
    const int v = sorted[t];
    pos[v] = base + t;
    visited[v] = 1;
    order[base + t] = v;
}
__global__ void k_rcm_degree(int n, const int* __restrict__ row_ptr, unsigned int* __restrict__ deg,
                             int* __restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    deg[i] = (unsigned int)(row_ptr[i + 1] - row_ptr[i]);
    idx[i] = i;
}
__global__ void k_rcm_start(int v, long long base, long long* __restrict__ pos, int* __restrict__ visited,
                            int* __restrict__ order, int* __restrict__ frontier) {
    pos[v] = base;
    visited[v] = 1;
    order[base] = v;
    frontier[0] = v;
}


// ---- greedy colouring (Jones-Plassmann) -------------------------------------
// Priority of node i: the high 32 bits of splitmix64(seed + i) above the node id, so every
// priority is distinct.  One round: an uncoloured node whose priority exceeds that of every
// uncoloured neighbour takes the smallest colour no coloured neighbour holds.  Colours are
// read from the previous round's array (double buffer): the result does not depend on
// thread timing, and mesh.py::greedy_colouring restates it exactly on the host.
__host__ __device__ inline unsigned long long jp_priority(int i, unsigned long long seed) {
    unsigned long long z = seed + (unsigned long long)(unsigned int)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (z & 0xFFFFFFFF00000000ull) | (unsigned long long)(unsigned int)i;
}
__global__ void k_jp_round(int n, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                           unsigned long long seed, const int* __restrict__ colour, int* __restrict__ colour_next,
                           int* __restrict__ remaining, int* __restrict__ overflow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ci_ = colour[i];
    if (ci_ >= 0) {
        colour_next[i] = ci_;
        return;
    }
    const unsigned long long pi = jp_priority(i, seed);
    unsigned long long used = 0;
    bool top = true;
    for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        const int j = col_idx[e];
        if (j == i) continue;
        const int cj = colour[j];
        if (cj >= 0) {
            if (cj < 64) used |= 1ull << cj;
        } else if (jp_priority(j, seed) > pi) {
            top = false;
        }
    }
    if (top) {
        const int c = __ffsll((long long)~used) - 1;
        if (c < 0) atomicExch(overflow, 1);
        colour_next[i] = c < 0 ? 63 : c;
    } else {
        colour_next[i] = -1;
        atomicAdd(remaining, 1);
    }
}
}  // namespace fnlh

using namespace fnlh;

struct fnlh_sector_dual {
    SectorDual d;
};

extern "C" {

int fnlh_sector_dual_create(int ci, int cj, int ck, int periodic_j, int tets, const double* Xu, long long* n_edges,
                            fnlh_sector_dual** out) {
    return guarded([&] {
        if (ci < 1 || cj < 1 || ck < 1) throw ConfigError("sector: cell counts must be >= 1");
        Dims d{};
        d.ci = ci;
        d.cj = cj;
        d.ck = ck;
        d.nju = cj + 1;
        d.nj = periodic_j ? cj : cj + 1;
        d.nk = ck + 1;
        d.periodic = periodic_j ? 1 : 0;
        d.ncell = (long long)ci * cj * ck;
        d.n = (long long)(ci + 1) * d.nj * d.nk;
        const long long nu = (long long)(ci + 1) * d.nju * d.nk;
        const Tables t = make_tables();
        const long long m = d.ncell * (tets ? 36 : 12);
        auto h = std::make_unique<fnlh_sector_dual>();
        SectorDual& s = h->d;
        s.n = d.n;
        cudaStream_t st = 0;
        DeviceBuffer<double> X, vecs((std::size_t)m * 3), vc((std::size_t)d.ncell * (tets ? 6 : 1));
        DeviceBuffer<unsigned long long> keys(m), keys_s(m);
        DeviceBuffer<long long> pos(m), pos_s(m), seg(m);
        DeviceBuffer<int> head(m);
        X.upload(Xu, (std::size_t)nu * 3);
        note_launch();
        if (tets)
            k_tet_cells<<<nb(d.ncell), kT, 0, st>>>(d, t, X.ptr, keys.ptr, vecs.ptr, vc.ptr);
        else
            k_hex_cells<<<nb(d.ncell), kT, 0, st>>>(d, t, X.ptr, keys.ptr, vecs.ptr, vc.ptr);
        FNLH_CUDA(cudaGetLastError());
        s.vol.alloc(d.n);
        note_launch();
        k_node_vol<<<nb(d.n), kT, 0, st>>>(d, t, tets, vc.ptr, s.vol.ptr);
        note_launch();
        k_iota<<<nb(m), kT, 0, st>>>(m, pos.ptr);
        // stable LSD radix sort: equal keys keep ascending positions (np.unique + bincount order)
        std::size_t tmp_bytes = 0;
        const int bits = key_bits(d.n);
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.ptr, keys_s.ptr, pos.ptr, pos_s.ptr, m, 0,
                                                  bits, st));
        DeviceBuffer<unsigned char> tmp(tmp_bytes);
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tmp_bytes, keys.ptr, keys_s.ptr, pos.ptr, pos_s.ptr, m, 0,
                                                  bits, st));
        note_launch();
        k_heads<<<nb(m), kT, 0, st>>>(m, keys_s.ptr, head.ptr);
        std::size_t tmp2 = 0;
        FNLH_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp2, head.ptr, seg.ptr, m, st));
        DeviceBuffer<unsigned char> tmpb(tmp2);
        FNLH_CUDA(cub::DeviceScan::InclusiveSum(tmpb.ptr, tmp2, head.ptr, seg.ptr, m, st));
        long long nuq = 0;
        FNLH_CUDA(cudaMemcpyAsync(&nuq, seg.ptr + (m - 1), sizeof nuq, cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
        DeviceBuffer<long long> start(nuq);
        note_launch();
        k_starts<<<nb(m), kT, 0, st>>>(m, head.ptr, seg.ptr, start.ptr);
        s.ne = nuq;
        s.ea.alloc(nuq);
        s.eb.alloc(nuq);
        s.en.alloc((std::size_t)nuq * 3);
        note_launch();
        k_edge_sums<<<nb(nuq), kT, 0, st>>>(nuq, m, d.n, start.ptr, keys_s.ptr, pos_s.ptr, vecs.ptr, s.ea.ptr, s.eb.ptr,
                                            s.en.ptr);
        FNLH_CUDA(cudaGetLastError());
        FNLH_CUDA(cudaStreamSynchronize(st));
        *n_edges = nuq;
        *out = h.release();
    });
}

int fnlh_sector_dual_get(const fnlh_sector_dual* h, long long* ea, long long* eb, double* en, double* vol) {
    return guarded([&] {
        const SectorDual& s = h->d;
        if (ea) download(ea, s.ea.ptr, s.ne);
        if (eb) download(eb, s.eb.ptr, s.ne);
        if (en) download(en, s.en.ptr, (std::size_t)s.ne * 3);
        if (vol) download(vol, s.vol.ptr, s.n);
    });
}

void fnlh_sector_dual_destroy(fnlh_sector_dual* h) { delete h; }

int fnlh_make_pattern(int rows, long long n_edges, const int* ea, const int* eb, int* row_ptr, int* col_idx,
                      int* diag_idx, long long* nnzb) {
    return guarded([&] {
        if (rows < 1) throw ShapeError("make_pattern: rows must be >= 1");
        cudaStream_t st = 0;
        const long long m = rows + 2 * n_edges;
        DeviceBuffer<int> a, c, bad(1), rp(rows + 1), ci(m), di(rows), nsel(1);
        DeviceBuffer<long long> nsel64(1);
        if (n_edges) {
            a.upload(ea, n_edges);
            c.upload(eb, n_edges);
        }
        FNLH_CUDA(cudaMemset(bad.ptr, 0, sizeof(int)));
        FNLH_CUDA(cudaMemset(di.ptr, 0xff, rows * sizeof(int)));
        DeviceBuffer<unsigned long long> keys(m), ks(m), uq(m);
        note_launch();
        k_pattern_keys<<<nb(std::max<long long>(rows, n_edges)), kT, 0, st>>>(rows, n_edges, a.ptr, c.ptr, keys.ptr,
                                                                              bad.ptr);
        int hbad = 0;
        FNLH_CUDA(cudaMemcpy(&hbad, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost));
        if (hbad) throw ShapeError("make_pattern: edge endpoint out of range");
        const int bits = key_bits(rows);
        std::size_t tb = 0;
        FNLH_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.ptr, ks.ptr, m, 0, bits, st));
        DeviceBuffer<unsigned char> tmp(tb);
        FNLH_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tb, keys.ptr, ks.ptr, m, 0, bits, st));
        std::size_t tu = 0;
        FNLH_CUDA(cub::DeviceSelect::Unique(nullptr, tu, ks.ptr, uq.ptr, nsel64.ptr, m, st));
        DeviceBuffer<unsigned char> tmpu(tu);
        FNLH_CUDA(cub::DeviceSelect::Unique(tmpu.ptr, tu, ks.ptr, uq.ptr, nsel64.ptr, m, st));
        long long nnz = 0;
        FNLH_CUDA(cudaMemcpyAsync(&nnz, nsel64.ptr, sizeof nnz, cudaMemcpyDeviceToHost, st));
        FNLH_CUDA(cudaStreamSynchronize(st));
        note_launch();
        k_pattern_fill<<<nb(nnz), kT, 0, st>>>(nnz, rows, uq.ptr, rp.ptr, ci.ptr, di.ptr);
        FNLH_CUDA(cudaGetLastError());
        download(row_ptr, rp.ptr, (std::size_t)rows + 1);
        download(col_idx, ci.ptr, (std::size_t)nnz);
        download(diag_idx, di.ptr, (std::size_t)rows);
        *nnzb = nnz;
    });
}

int fnlh_rcm(int n, const int* row_ptr, const int* col_idx, const int* starts, int* perm) {
    return guarded([&] {
        if (n < 1) throw ShapeError("rcm: n must be >= 1");
        for (int i = 0; i < n; ++i)
            if (row_ptr[i + 1] - row_ptr[i] > 255) throw ShapeError("rcm: degree above 255");
        cudaStream_t st = 0;
        const long long nnz = row_ptr[n];
        DeviceBuffer<int> rp, ci, visited(n), mark(n), order(n), frontier(n), next(n), sorted(n), nnext(1), idx(n),
            idx_s(n);
        DeviceBuffer<long long> pos(n);
        DeviceBuffer<unsigned long long> claim(n), keys(n), keys_s(n);
        DeviceBuffer<unsigned int> deg(n), deg_s(n);
        rp.upload(row_ptr, (std::size_t)n + 1);
        ci.upload(col_idx, (std::size_t)nnz);
        FNLH_CUDA(cudaMemset(visited.ptr, 0, n * sizeof(int)));
        FNLH_CUDA(cudaMemset(mark.ptr, 0, n * sizeof(int)));
        FNLH_CUDA(cudaMemset(claim.ptr, 0xff, n * sizeof(unsigned long long)));
        // component starts: nodes by ascending degree, stable (scipy's argsort of degrees)
        note_launch();
        k_rcm_degree<<<nb(n), kT, 0, st>>>(n, rp.ptr, deg.ptr, idx.ptr);
        std::size_t tb = 0, tb2 = 0;
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, deg.ptr, deg_s.ptr, idx.ptr, idx_s.ptr, n, 0, 9, st));
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, keys.ptr, keys_s.ptr, next.ptr, sorted.ptr, n, 0, 64, st));
        DeviceBuffer<unsigned char> tmp(std::max(tb, tb2));
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, deg.ptr, deg_s.ptr, idx.ptr, idx_s.ptr, n, 0, 9, st));
        std::vector<int> by_deg(n), vis(n);
        if (starts) {  // the caller's seed order (scipy: np.argsort(degree), an unstable sort)
            std::copy(starts, starts + n, by_deg.begin());
        } else {
            FNLH_CUDA(cudaMemcpyAsync(by_deg.data(), idx_s.ptr, n * sizeof(int), cudaMemcpyDeviceToHost, st));
            FNLH_CUDA(cudaStreamSynchronize(st));
        }
        const int kbits = 64;
        long long base = 0;
        std::size_t cursor = 0;
        while (base < n) {
            FNLH_CUDA(cudaMemcpyAsync(vis.data(), visited.ptr, n * sizeof(int), cudaMemcpyDeviceToHost, st));
            FNLH_CUDA(cudaStreamSynchronize(st));
            while (vis[by_deg[cursor]]) ++cursor;
            note_launch();
            k_rcm_start<<<1, 1, 0, st>>>(by_deg[cursor], base, pos.ptr, visited.ptr, order.ptr, frontier.ptr);
            ++base;
            int nf = 1;
            while (nf > 0) {
                FNLH_CUDA(cudaMemsetAsync(nnext.ptr, 0, sizeof(int), st));
                note_launch();
                k_rcm_claim<<<nb(nf), kT, 0, st>>>(nf, frontier.ptr, pos.ptr, rp.ptr, ci.ptr, visited.ptr, claim.ptr,
                                                   mark.ptr, next.ptr, nnext.ptr);
                int nn = 0;
                FNLH_CUDA(cudaMemcpyAsync(&nn, nnext.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
                FNLH_CUDA(cudaStreamSynchronize(st));
                if (nn == 0) break;
                note_launch();
                k_rcm_keys<<<nb(nn), kT, 0, st>>>(nn, next.ptr, claim.ptr, rp.ptr, keys.ptr);
                std::size_t tbl = tb2;
                FNLH_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tbl, keys.ptr, keys_s.ptr, next.ptr, sorted.ptr, nn,
                                                          0, kbits, st));
                note_launch();
                k_rcm_assign<<<nb(nn), kT, 0, st>>>(nn, sorted.ptr, base, pos.ptr, visited.ptr, order.ptr);
                base += nn;
                std::swap(frontier.ptr, sorted.ptr);
                nf = nn;
            }
        }
        std::vector<int> cm(n);
        download(cm.data(), order.ptr, (std::size_t)n);
        for (int i = 0; i < n; ++i) perm[i] = cm[n - 1 - i];  // reversed: perm[position] = node
    });
}

int fnlh_mesh_derive(int n, int nf, const int* fa, const int* fb, const double* fn, const double* coords,
                     double* farea, double* fnh, double* fvis, int* nf_ptr, int* nf_idx, double* closure, int* bflag) {
    return guarded([&] {
        cudaStream_t st = 0;
        const long long m = 2LL * nf;
        DeviceBuffer<int> dfa, dfb, ev(m), ev_s(m), np(n + 1), nidx(m), bf(n);
        DeviceBuffer<double> dfn, X, fa_(nf), fnh_(3LL * nf), fv_(nf), cl(3LL * n);
        DeviceBuffer<unsigned int> node(m), node_s(m);
        dfa.upload(fa, nf);
        dfb.upload(fb, nf);
        dfn.upload(fn, 3LL * nf);
        if (coords) X.upload(coords, 3LL * n);
        note_launch();
        k_face_events<<<nb(nf), kT, 0, st>>>(nf, dfa.ptr, dfb.ptr, node.ptr, ev.ptr);
        // stable sort by node: each node's faces stay in ascending face order
        std::size_t tb = 0;
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, node.ptr, node_s.ptr, ev.ptr, ev_s.ptr, m, 0, 32, st));
        DeviceBuffer<unsigned char> tmp(tb);
        FNLH_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, node.ptr, node_s.ptr, ev.ptr, ev_s.ptr, m, 0, 32, st));
        FNLH_CUDA(cudaMemsetAsync(np.ptr, 0, (n + 1) * sizeof(int), st));
        note_launch();
        k_node_ptr<<<nb(m), kT, 0, st>>>(m, n, node_s.ptr, np.ptr);
        note_launch();
        k_face_derived<<<nb(nf), kT, 0, st>>>(nf, dfn.ptr, dfa.ptr, dfb.ptr, coords ? X.ptr : nullptr, fa_.ptr,
                                              fnh_.ptr, fv_.ptr);
        note_launch();
        k_node_derived<<<nb(n), kT, 0, st>>>(n, np.ptr, ev_s.ptr, dfn.ptr, dfb.ptr, nidx.ptr, cl.ptr, bf.ptr);
        FNLH_CUDA(cudaGetLastError());
        FNLH_CUDA(cudaStreamSynchronize(st));
        int total = 0;
        FNLH_CUDA(cudaMemcpy(&total, np.ptr + n, sizeof(int), cudaMemcpyDeviceToHost));
        download(farea, fa_.ptr, nf);
        download(fnh, fnh_.ptr, 3LL * nf);
        download(fvis, fv_.ptr, nf);
        download(nf_ptr, np.ptr, (std::size_t)n + 1);
        download(nf_idx, nidx.ptr, (std::size_t)total);
        download(closure, cl.ptr, 3LL * n);
        download(bflag, bf.ptr, n);
    });
}

int fnlh_greedy_colour(int n, const int* row_ptr, const int* col_idx, unsigned long long seed, int* colour,
                       int* ncolours) {
    return guarded([&] {
        if (n < 1) throw ShapeError("greedy_colour: n must be >= 1");
        const long long nnz = row_ptr[n];
        DeviceBuffer<int> rp, ci, c0(n), c1(n), rem(1), ovf(1);
        rp.upload(row_ptr, (std::size_t)n + 1);
        ci.upload(col_idx, (std::size_t)nnz);
        FNLH_CUDA(cudaMemset(c0.ptr, 0xff, n * sizeof(int)));
        FNLH_CUDA(cudaMemset(ovf.ptr, 0, sizeof(int)));
        int left = n, rounds = 0;
        while (left > 0) {
            FNLH_CUDA(cudaMemset(rem.ptr, 0, sizeof(int)));
            note_launch();
            k_jp_round<<<nb(n), kT>>>(n, rp.ptr, ci.ptr, seed, c0.ptr, c1.ptr, rem.ptr, ovf.ptr);
            FNLH_CUDA(cudaGetLastError());
            std::swap(c0.ptr, c1.ptr);
            FNLH_CUDA(cudaMemcpy(&left, rem.ptr, sizeof(int), cudaMemcpyDeviceToHost));
            if (++rounds > n) throw std::runtime_error("greedy_colour: no progress");
        }
        int over = 0;
        FNLH_CUDA(cudaMemcpy(&over, ovf.ptr, sizeof(int), cudaMemcpyDeviceToHost));
        if (over) throw UnsupportedCaseError("greedy_colour: more than 64 colours");
        download(colour, c0.ptr, (std::size_t)n);
        int mx = -1;
        for (int i = 0; i < n; ++i) mx = std::max(mx, colour[i]);
        *ncolours = mx + 1;
    });
}

}  // extern "C"
