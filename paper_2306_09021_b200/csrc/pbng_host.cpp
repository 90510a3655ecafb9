// pbng_host.cpp -- host side of libpbng: the C ABI of include/pbng.h.
//
// Owns validation, the fp64 rest-state precompute, Lame conversion (eq:lame), the
// greedy node colouring, the colour-sorted SELL-32 device layout, the workspace plan
// and the launch sequence of PBNG iterations.  Every per-iteration arithmetic step
// runs in the kernels of pbng_kernels.cu; there is no CPU fallback.
#include "pbng.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <thread>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "pbng_internal.h"

using namespace pbng;

namespace {

thread_local std::string g_err = "no error";

// PBNG_TIMING=1: host phase timings of the constraint-update path on stderr (tools/contact_timing.py)
struct PhaseTimer {
    bool on;
    std::chrono::steady_clock::time_point t0;
    PhaseTimer() : on(getenv("PBNG_TIMING") && atoi(getenv("PBNG_TIMING")) != 0), t0(std::chrono::steady_clock::now()) {}
    void lap(const char *what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[pbng] %-32s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

pbng_status fail(pbng_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

pbng_status cuda_fail(cudaError_t e, const char *where) {
    return fail(PBNG_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define PBNG_CUDA(call, where)                          \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

struct DevGuard {
    int prev = -1, dev = -1;
    explicit DevGuard(int d) : dev(d) {
        if (d >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
    }
    ~DevGuard() {
        if (dev >= 0 && prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// fn(lo, hi) over [0, n) in contiguous blocks on up to 16 host threads (independent iterations only; the
// result must not depend on the split -- every caller writes disjoint outputs per index)
template <class F>
void parallel_for(int64_t n, F &&fn, int64_t min_per_thread = 4096) {
    const int64_t hw = std::max<int64_t>(1, std::min<int64_t>(16, (int64_t)std::thread::hardware_concurrency()));
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hw, n / std::max<int64_t>(min_per_thread, 1)));
    if (nt <= 1) {
        fn((int64_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int64_t k = 0; k < nt; ++k) th.emplace_back([&, k] { fn(n * k / nt, n * (k + 1) / nt); });
    for (auto &t : th) t.join();
}

double det3(const double *M) {
    return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
           M[2] * (M[3] * M[7] - M[4] * M[6]);
}

// Chebyshev weights: omega_m = 1 (m <= 2), 2/(2-rho^2) (m = 3), 4/(4 - rho^2 omega_{m-1})
double chebyshev_weight(int64_t m, double rho) {
    if (m <= 2) return 1.0;
    double w = 2.0 / (2.0 - rho * rho);
    for (int64_t k = 4; k <= m; ++k) w = 4.0 / (4.0 - rho * rho * w);
    return w;
}

struct Region {
    size_t off = 0, bytes = 0;
};

// 3 x 21-bit Morton (Z-order) interleave
uint64_t spread21(uint64_t x) {
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}
uint64_t morton3(uint64_t a, uint64_t b, uint64_t c) { return spread21(a) | spread21(b) << 1 | spread21(c) << 2; }

// sample-minor position layout for large batches (the batched sweep kernel); PBNG_BATCHED=0 disables
bool batched_layout(const pbng_ctx *c);

// intra-colour vertex order: Morton (default) or ascending index (PBNG_ORDER=index, for experiments)
bool spatial_order() {
    const char *e = getenv("PBNG_ORDER");
    return !(e && std::string(e) == "index");
}

}  // namespace

struct pbng_ctx {
    // mesh
    int64_t nv = 0, nt = 0;
    int32_t nb = 1;
    int dtype = DT_F32;
    int device = -1;
    cudaStream_t stream = nullptr;
    std::vector<double> X;
    std::vector<int32_t> tets;
    std::vector<double> Bm;  // per tet Dm^{-1} (row-major)
    std::vector<double> V;   // per tet rest volume
    // material
    bool has_material = false;
    int model = MODEL_NH;
    std::vector<double> E;
    double nu = 0, density = 0, grav[3] = {0, 0, 0};
    // constraints
    bool has_constraints = false;
    std::vector<int32_t> pinned;   // ascending
    std::vector<double> targets;   // [nb][npin][3] in ascending pinned order
    std::vector<pbng_weak_constraint> wc;
    // domain decomposition (pbng_set_partition); an empty owner list means one rank owns everything
    std::vector<int32_t> owner;
    int32_t rank = 0, n_ranks = 1;
    // colouring + layout.  Local vertex order: owned free (colour-major) | ghost free | held pinned.
    bool colored = false;
    std::vector<int32_t> colour;
    int32_t ncol = 0;
    std::vector<int32_t> orig2int, int2orig;  // orig2int = -1 for vertices this context does not hold
    int64_t n_free = 0;        // owned free vertices (the swept set)
    int64_t n_local_free = 0;  // owned + ghost free vertices
    int64_t n_local = 0;       // all held vertices
    int64_t n_pairs = 0, n_slots = 0, n_chunks = 0, n_vc = 0;
    std::vector<int32_t> local_pinned;  // indices into `pinned` of the held pinned vertices
    std::vector<int32_t> tet_local;     // tets whose energy this context evaluates (owner of vertex 0)
    std::vector<int32_t> cons_local;    // constraints held: owned ones (energy) first, then the others
    int64_t n_cons_owned = 0;
    std::vector<int64_t> halo_send_off, halo_recv_off;  // [ncol * n_ranks + 1]
    std::vector<int32_t> h_halo_send, h_halo_recv;      // internal ids, ascending original index
    std::vector<int32_t> halo_send_orig, halo_recv_orig;  // the same lists as original vertex ids
    int cur_accel = -1;  // acceleration of the colour passes of the iteration in progress (-1: none yet)
    std::vector<int32_t> col_vbegin, col_nfree;
    std::vector<int32_t> col_nsend;   // per colour: owned free vertices some other rank holds (laid out first)
    std::vector<int64_t> col_chunk_mid;  // per colour: first chunk of the vertices after the halo-send ones
    std::vector<int64_t> gcol_nfree;  // free vertices per colour over the whole mesh (all ranks)
    std::vector<int64_t> col_chunk;
    // host images of the device arrays (uploaded by bind)
    std::vector<int4> h_rec_id;
    std::vector<int2> h_rec_id2;   // path-ordered NH records: {id | drop << 30, VE bits} (Problem::path)
    std::vector<int2> h_path0;     // path-ordered NH records: per free vertex the slots S1, S2 before record 0
    bool path_rec = false;
    // rest-recompute path records (SURVEY.md §8(d) lower-byte variant (i)): {id | drop, E_e/6} only, the
    // kernels rebuild s'_j, det B' and V_e from the rest positions h_rest (Real4 [n_local], internal ids)
    bool rest_rec = false;
    // table path records: h_rec_a holds the n_tab distinct {s'_0..2, det B'} tuples, record codes index them
    bool tab_rec = false;
    int64_t n_tab = 0;
    int records = 0;  // pbng_records requested (0 auto, 1 stored rest data, 2 rest recompute, 3 table)
    std::vector<unsigned char> h_rest;
    std::vector<int64_t> inc_off;  // vertex -> incident tets (ascending), mesh-only: built once and kept
    std::vector<int32_t> inc;
    void *stage2 = nullptr;  // second staging buffer (device re-layout of pbng_update_constraints)
    size_t wc_cap = 0, vc_cap = 0, deps_cap = 0;  // weak-constraint / pipeline-dependency room in the workspace
    int64_t n_records = 0;         // pair records stored per sweep (path mode: incl. load-only ones)
    std::vector<unsigned char> h_rec_a, h_rec_b, h_rec_c, h_fext, h_wc_d, h_c_w, h_c_anchor, h_c_K, h_tet_a,
        h_tet_b, h_tet_c, h_targets;
    std::vector<int64_t> h_chunk_off;
    std::vector<int2> h_chunk_v;
    std::vector<int32_t> h_deg, h_wc_off, h_wc_cid, h_c_n, h_c_node;
    std::vector<unsigned char> h_mass;  // Real [n_own] lumped masses (backward Euler)
    std::vector<int32_t> h_dep_off, h_deps;  // pipelined schedule: per chunk its neighbour chunks (Layout)
    // contact detection (pbng_detect_contacts): boundary triangles {v0, v1, v2, body} and the free boundary
    // vertices {vertex, body}, internal ids; tri_orig = the triangles' original vertex ids
    std::vector<int4> h_surf;
    std::vector<int2> h_sv;
    std::vector<int32_t> surf_orig;                  // boundary triangles in original ids (mesh-only, cached)
    std::vector<int32_t> surf_body, surf_verts, surf_vbody;  // per triangle body; boundary vertices and bodies
    bool surf_cached = false;
    std::vector<int64_t> pin_order;  // caller order of the pinned set -> ascending order (set_constraints)
    uint64_t ws_bytes = 0;           // bytes of the bound workspace
    bool l2_persist = false;         // pbng_set_l2_persistence (re-applied by every bind)
    // state the library changed outside its own memory while the L2 window is on, restored by
    // clear_l2_persistence (pbng_destroy, set_stream, disabling): the stream that carries the window and
    // the device's persisting-L2 limit before the library set it
    bool l2_applied = false;
    cudaStream_t l2_stream = nullptr;
    size_t l2_prev_limit = 0;
    int schedule = 0;                        // pbng_schedule requested (0 auto, 1 colour launches, 2 pipelined)
    std::vector<int4> h_tet_id;
    Problem prob;
    // workspace plan
    Region r_rec_id, r_rec_a, r_rec_b, r_rec_c, r_chunk_off, r_chunk_v, r_deg, r_fext, r_wc_off, r_wc_cid, r_wc_d,
        r_c_n, r_c_node, r_c_w, r_c_anchor, r_c_K, r_tet_id, r_tet_a, r_tet_b, r_tet_c, r_int2orig, r_targets,
        r_x[3], r_stage, r_part_e, r_part_r, r_results, r_flag, r_halo_send, r_halo_recv, r_mass, r_xt, r_dep_off,
        r_deps, r_pipe, r_surf, r_sv, r_chead, r_cnext, r_cres, r_cscal, r_hsend, r_hrecv, r_allred, r_path0, r_stage2,
        r_rest;
    size_t ws_need = 0;
    // bound device state
    bool bound = false;
    void *ws = nullptr;
    Layout L;
    bool positions_set = false;
    int work = 0, out = 1, hist = 2;
    int64_t l = 0;
    bool hist_valid = true;
    int64_t launches = 0;
    // in-library halo transport (pbng_partition / pbng_group_*): NCCL communicator, the side stream that
    // carries pack -> exchange -> unpack, fork/join events, and the CUDA graph of the last iterate block
    ncclComm_t comm = nullptr;
    cudaStream_t dd_side = nullptr, dd_cap = nullptr;
    cudaEvent_t dd_ev_a = nullptr, dd_ev_b = nullptr;
    struct GraphKey {
        int32_t n = -1;
        int accel = -1;
        double omega = 0, rho = 0, gamma = 0;
        int64_t l = -1;
        int work = -1, out = -1, hist = -1;
        bool hist_valid = false;
        const void *ws = nullptr;
        cudaStream_t stream = nullptr;
        double inv_dt2 = -1;
        std::vector<uint64_t> gens;  // layout generation of every rank context the block drives
        bool operator==(const GraphKey &o) const {
            return n == o.n && accel == o.accel && omega == o.omega && rho == o.rho && gamma == o.gamma && l == o.l &&
                   work == o.work && out == o.out && hist == o.hist && hist_valid == o.hist_valid && ws == o.ws &&
                   stream == o.stream && inv_dt2 == o.inv_dt2 && gens == o.gens;
        }
    } dd_key;
    uint64_t layout_gen = 0;  // bumped by every re-layout / bind: captured launches bake the layout in
    // peer-store halo transport (pbng_enable_peer_halo / pbng_group_set_transport): the neighbours' position
    // buffers and flag words through peer mappings, this rank's own flag words and the neighbours' ghost rows
    struct PeerState {
        bool enabled = false;
        uint64_t gen = 0;          // layout_gen and workspace the mappings were made for
        const void *ws = nullptr;
        uint32_t *flags = nullptr;  // own allocation: pushed[n_ranks] | done[n_ranks] | counter[n_ranks] | scratch[4]
        int32_t *rows = nullptr;    // [halo_send_off.back()] the send vertices' ghost rows on their receiver
        std::vector<int> nbr;       // ranks this one exchanges any row with
        struct Peer {
            void *x[3] = {nullptr, nullptr, nullptr};
            int64_t stride = 0;
            int sh = 0;
            int64_t n_local = 0;  // vertices the neighbour holds
            uint32_t *flags = nullptr;
            void *ipc_ws = nullptr, *ipc_flags = nullptr;  // cudaIpcOpenMemHandle results (multi-process)
        };
        std::vector<Peer> peer;  // [n_ranks]
    } peer;
    cudaGraphExec_t dd_graph = nullptr;
    int64_t dd_graph_launches = 0;   // kernels one replay of dd_graph runs
    int64_t dd_graph_sweeps = 0;     // sweep launches one replay of dd_graph runs
    int64_t dd_graph_replays = 0;    // replays since creation (tests: the cache is used)
    // profiling
    int profiling = 0;  // 0 off, 1 per sweep launch, 2 per iterate span (back-to-back sweep launches)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used, ev_free;
    std::vector<int64_t> ev_launches;

    size_t real_size() const { return dtype == DT_F64 ? 8 : 4; }
    size_t real4_size() const { return dtype == DT_F64 ? 32 : 16; }
    bool on_device() const { return device >= 0; }

    ~pbng_ctx() {
        for (auto &e : ev_used) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
        for (auto &e : ev_free) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    }

    void invalidate_colouring() {
        colored = false;
        bound = false;
        positions_set = false;
    }
};

namespace {

// ------------------------------------------------------------------------------------------------
// typed writers for the host images
// ------------------------------------------------------------------------------------------------
template <class R>
void put4(std::vector<unsigned char> &buf, int64_t idx, double a, double b, double c, double d) {
    R *p = reinterpret_cast<R *>(buf.data()) + 4 * idx;
    p[0] = R(a); p[1] = R(b); p[2] = R(c); p[3] = R(d);
}

template <class R>
void put1(std::vector<unsigned char> &buf, int64_t idx, double a) {
    reinterpret_cast<R *>(buf.data())[idx] = R(a);
}

// gradient of local node k of tet e (k >= 1: row k-1 of Dm^{-1}; k = 0: minus the row sum)
inline void shape_grad(const pbng_ctx *c, int64_t e, int k, double g[3]) {
    const double *B = c->Bm.data() + 9 * e;
    for (int b = 0; b < 3; ++b) g[b] = k > 0 ? B[3 * (k - 1) + b] : -(B[b] + B[3 + b] + B[6 + b]);
}

// ------------------------------------------------------------------------------------------------
// greedy node colouring, PAPER.md:702-705 (library implementation: 64-bit used-colour masks per
// stencil; vertices in ascending index; colour = least colour not used by any stencil of the vertex)
// ------------------------------------------------------------------------------------------------
pbng_status colour_greedy(pbng_ctx *c, const std::vector<int64_t> &vs_off, const std::vector<int64_t> &vs) {
    const int64_t n_st = c->nt + (int64_t)c->wc.size();
    for (int W = 1;; W *= 2) {
        std::vector<uint64_t> used((size_t)n_st * W, 0ull);
        std::vector<uint64_t> forb(W);
        bool overflow = false;
        int32_t maxc = 0;
        for (int64_t v = 0; v < c->nv && !overflow; ++v) {
            std::fill(forb.begin(), forb.end(), 0ull);
            for (int64_t k = vs_off[v]; k < vs_off[v + 1]; ++k) {
                const uint64_t *u = used.data() + (size_t)vs[k] * W;
                for (int w = 0; w < W; ++w) forb[w] |= u[w];
            }
            int32_t col = -1;
            for (int w = 0; w < W && col < 0; ++w)
                if (~forb[w]) col = 64 * w + __builtin_ctzll(~forb[w]);
            if (col < 0) { overflow = true; break; }
            c->colour[v] = col;
            maxc = std::max(maxc, col + 1);
            for (int64_t k = vs_off[v]; k < vs_off[v + 1]; ++k)
                used[(size_t)vs[k] * W + col / 64] |= 1ull << (col % 64);
        }
        if (!overflow) {
            c->ncol = maxc;
            return PBNG_OK;
        }
        if (W > 1024) return fail(PBNG_E_INVALID_ARGUMENT, "colouring needs more than 65536 colours");
    }
}

// ------------------------------------------------------------------------------------------------
// Path-ordered Neo-Hookean records.  PAPER.md:697-705 leaves each vertex free to sum its incident tets in
// any order; the library orders them along paths in the dual graph of the vertex's link (the triangles
// opposite the vertex, adjacent when two tets share a face through it, i.e. two of their three other
// vertices).  Consecutive records then share two neighbours, so the kernel keeps three position slots in
// registers and gathers ONE new neighbour per record instead of three (pbng_kernels.cu "path records").
// Greedy Warnsdorff cover (next = the unused adjacent triangle with the fewest unused neighbours), retried
// with seeded tie-breaking while it needs more than one path; Kuhn-grid links take one path per vertex.
// ------------------------------------------------------------------------------------------------
void link_paths(const std::vector<std::array<int32_t, 3>> &tri, uint32_t seed, std::vector<std::vector<int>> &best) {
    const int n = (int)tri.size();
    std::vector<std::vector<int>> adj(n);
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b) {
            int sh = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) sh += tri[a][i] == tri[b][j];
            if (sh == 2) {
                adj[a].push_back(b);
                adj[b].push_back(a);
            }
        }
    best.clear();
    uint32_t rng = seed * 2654435761u + 12345u;
    std::vector<char> used(n);
    std::vector<int> free_deg(n);
    std::vector<std::vector<int>> paths;
    for (int trial = 0; trial < 24; ++trial) {
        std::fill(used.begin(), used.end(), 0);
        for (int k = 0; k < n; ++k) free_deg[k] = (int)adj[k].size();
        paths.clear();
        auto take = [&](int k) {
            used[k] = 1;
            for (int q : adj[k]) --free_deg[q];
        };
        auto pick = [&](const std::vector<int> &cand) {  // fewest unused neighbours; ties: first / seeded
            int bestk = -1, bd = 1 << 30, ties = 0;
            for (int k : cand) {
                if (used[k]) continue;
                if (free_deg[k] < bd) { bd = free_deg[k]; bestk = k; ties = 1; }
                else if (free_deg[k] == bd && trial > 0) {
                    ++ties;
                    rng = rng * 1664525u + 1013904223u;
                    if ((rng >> 8) % (uint32_t)ties == 0) bestk = k;
                }
            }
            return bestk;
        };
        std::vector<int> all(n);
        for (int k = 0; k < n; ++k) all[k] = k;
        for (int remaining = n; remaining > 0;) {
            int k = pick(all);
            std::vector<int> path;
            while (k >= 0) {
                take(k);
                path.push_back(k);
                --remaining;
                k = pick(adj[k]);
            }
            paths.push_back(path);
        }
        if (best.empty() || paths.size() < best.size()) best = paths;
        if (best.size() <= 1) break;
    }
}

// records of NH pair k of a vertex in path order: `tet` = index into the vertex's incident-tet list (-1:
// load-only), `vnew` the neighbour pushed, `drop` the slot code, `slot` the slot contents after the push
struct PathRec {
    int tet;
    int32_t vnew;
    int drop;
    int32_t slot[3];
};
// Path covers depend only on the link's structure, so they are memoised per thread by a canonical key
// (vertex labels replaced by order of first appearance); the retry seed is a hash of that key, so the
// result is a pure function of the structure -- independent of thread count, memo state and vertex id.
struct PathMemo {
    std::unordered_map<std::string, std::vector<std::vector<int>>> m;
};
void vertex_path_records(const std::vector<std::array<int32_t, 3>> &tri, uint32_t /*unused*/, std::vector<PathRec> &out,
                         int32_t path0[2], PathMemo *memo = nullptr) {
    out.clear();
    std::string key;
    {
        std::vector<std::pair<int32_t, unsigned char>> seen;
        key.reserve(3 * tri.size());
        for (const auto &t : tri)
            for (int a = 0; a < 3; ++a) {
                unsigned char id = 0xff;
                for (const auto &pv : seen)
                    if (pv.first == t[a]) id = pv.second;
                if (id == 0xff) {
                    id = (unsigned char)std::min<size_t>(seen.size(), 0xfe);
                    seen.push_back({t[a], id});
                }
                key.push_back((char)id);
            }
    }
    uint32_t seed = 2166136261u;
    for (char ch : key) seed = (seed ^ (unsigned char)ch) * 16777619u;
    std::vector<std::vector<int>> paths;
    auto hit = memo && tri.size() <= 250 ? memo->m.find(key) : (memo ? memo->m.end() : decltype(memo->m.end())());
    if (memo && tri.size() <= 250 && hit != memo->m.end()) {
        paths = hit->second;
    } else {
        link_paths(tri, seed, paths);
        if (memo && tri.size() <= 250) memo->m.emplace(key, paths);
    }
    int32_t S[3] = {-1, -1, -1};
    auto push = [&](int tet, int32_t vnew, int drop) {
        if (drop == 2) S[2] = S[1];
        if (drop >= 1) S[1] = S[0];
        S[0] = vnew;
        out.push_back({tet, vnew, drop, {S[0], S[1], S[2]}});
    };
    for (size_t pi = 0; pi < paths.size(); ++pi) {
        const std::vector<int> &P = paths[pi];
        const std::array<int32_t, 3> &t0 = tri[P[0]];
        if (pi == 0) {  // the first triangle's other two vertices come from path0 (S1, S2 before record 0)
            path0[0] = S[1] = t0[1];
            path0[1] = S[2] = t0[2];
            push(P[0], t0[0], 0);
        } else {  // a further path: two load-only pushes, then the triangle itself
            push(-1, t0[0], 2);
            push(-1, t0[1], 2);
            push(P[0], t0[2], 2);
        }
        for (size_t q = 1; q < P.size(); ++q) {
            const std::array<int32_t, 3> &t = tri[P[q]];
            int drop = -1;
            int32_t vnew = -1;
            for (int sl = 0; sl < 3; ++sl)
                if (t[0] != S[sl] && t[1] != S[sl] && t[2] != S[sl]) drop = sl;
            for (int a = 0; a < 3; ++a)
                if (t[a] != S[0] && t[a] != S[1] && t[a] != S[2]) vnew = t[a];
            push(P[q], vnew, drop);
        }
    }
    if (paths.empty()) path0[0] = path0[1] = -1;
}

int problem_split(const pbng_ctx *c);
bool batched_layout(const pbng_ctx *c);

// PBNG_PATH=0 keeps the plain three-id NH records everywhere (experiments; fp32 NH batches then use the
// sample-minor sh-5 layout, since sweep_batched2_kernel reads path records only)
bool path_env() {
    static const int env = [] {
        const char *e = getenv("PBNG_PATH");
        return e ? atoi(e) : 1;
    }();
    return env != 0;
}

int layout_lane_shift(const pbng_ctx *c) {
    if (!batched_layout(c)) return 0;
    return (c->dtype == DT_F32 && c->model == MODEL_NH && path_env() && c->n_local < (1 << 30)) ? 6 : 5;
}

// path-ordered NH records for the kernels that walk a vertex's records in order on one lane or one warp:
// sweep_kernel with one warp per chunk (problem_split 1) and sweep_batched2_kernel (sh 6)
bool use_path_records(const pbng_ctx *c) {
    if (!path_env() || c->model != MODEL_NH || c->n_local >= (1 << 30)) return false;
    const int sh = layout_lane_shift(c);
    return sh == 6 || (sh == 0 && problem_split(c) == 1);
}

// rest-recompute records (pbng_records; PBNG_RECORDS=1|2 overrides auto for experiments): path records of
// the one-thread-per-vertex sweep only (sh 0).  The batched kernel shares each record across 64 samples
// of a warp, so its records cost no HBM per sample and recomputing them per lane would only add ALU work.
bool use_rest_records(const pbng_ctx *c) {
    static const int env = [] {
        const char *e = getenv("PBNG_RECORDS");
        return e ? atoi(e) : 0;
    }();
    if (!c->path_rec || layout_lane_shift(c) != 0) return false;
    const int want = c->records != 0 ? c->records : env;
    return want == 2;
}

// table records: wanted when requested (pbng_records 3 / PBNG_RECORDS=3) or by auto, for the same contexts
// as the rest-recompute ones and ids below 2^22 (bits 22..29 of the code carry the table index); whether the
// mesh has few enough distinct rest tuples is only known once the records exist (build_rest_table)
bool want_table_records(const pbng_ctx *c) {
    static const int env = [] {
        const char *e = getenv("PBNG_RECORDS");
        return e ? atoi(e) : 0;
    }();
    if (!c->path_rec || layout_lane_shift(c) != 0 || c->n_local >= (1 << 22)) return false;
    const int want = c->records != 0 ? c->records : env;
    return want == 3 || want == 0;
}

// Table records are regrouped so that a lane's records come in groups of kRecGroup consecutive slots
// (pbng_kernels.cu update_vertex_path, mode 3): record k of lane `lane` of chunk ch sits at
//     chunk_off[ch] + (k / 4) * 128 + 4 * lane + k % 4,
// chunk widths rounded up to a multiple of 4 (padding slots: code 0, VE 0, never read), so one lane loads
// four 8-byte records with two 16-byte loads and has four neighbour gathers in flight at once.
template <class R>
void group_table_records(pbng_ctx *c) {
    const int64_t nch = c->n_chunks;
    std::vector<int64_t> off((size_t)nch + 1, 0);
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t w = (c->h_chunk_off[ch + 1] - c->h_chunk_off[ch]) / kChunk;
        off[ch + 1] = off[ch] + (w + kRecGroup - 1) / kRecGroup * kRecGroup * kChunk;
    }
    const bool f64 = c->dtype == DT_F64;
    std::vector<int2> id2((size_t)std::max<int64_t>(off[nch], 1), make_int2(0, 0));
    std::vector<unsigned char> rc(f64 ? (size_t)std::max<int64_t>(off[nch], 1) * 8 : c->h_rec_c.size(), 0);
    parallel_for(nch, [&](int64_t lo, int64_t hi) {
        for (int64_t ch = lo; ch < hi; ++ch) {
            const int64_t w = (c->h_chunk_off[ch + 1] - c->h_chunk_off[ch]) / kChunk;
            for (int64_t k = 0; k < w; ++k)
                for (int lane = 0; lane < kChunk; ++lane) {
                    const int64_t r = c->h_chunk_off[ch] + k * kChunk + lane;
                    const int64_t r2 = off[ch] + (k / kRecGroup) * (kRecGroup * kChunk) + kRecGroup * lane + k % kRecGroup;
                    id2[r2] = c->h_rec_id2[r];
                    if (f64) std::memcpy(rc.data() + r2 * 8, c->h_rec_c.data() + r * 8, 8);
                }
        }
    }, 256);
    c->h_rec_id2.swap(id2);
    if (f64) c->h_rec_c.swap(rc);
    c->h_chunk_off.swap(off);
    c->n_slots = c->h_chunk_off.back();
}

// Deduplicate the stored path records' rest data {s'_0..2, det B'} (compared bit for bit in the compute
// dtype) into a table of at most 256 entries; on success h_rec_a becomes the table and each record's code
// carries its entry in bits 22..29, so the kernels read exactly the values the stored layout holds.
// Regular meshes (the configs' Kuhn grids, the paper's 5-tet grids) repeat a few element shapes; an
// irregular mesh overflows the table and keeps the stored layout.
template <class R>
bool build_rest_table(pbng_ctx *c) {
    constexpr size_t K = 4 * sizeof(R);
    struct Key {
        unsigned char b[K];
        bool operator==(const Key &o) const { return std::memcmp(b, o.b, K) == 0; }
    };
    struct Hash {
        size_t operator()(const Key &k) const {
            uint64_t h = 1469598103934665603ull;
            for (size_t q = 0; q < K; ++q) h = (h ^ k.b[q]) * 1099511628211ull;
            return (size_t)h;
        }
    };
    const int64_t ns = c->n_slots;
    if (ns <= 0) return false;
    auto key_at = [&](int64_t r) {
        Key k;
        std::memcpy(k.b, c->h_rec_a.data() + (size_t)r * K, K);
        return k;
    };
    std::unordered_map<Key, int32_t, Hash> table;
    std::mutex mu;
    bool overflow = false;
    parallel_for(ns, [&](int64_t lo, int64_t hi) {
        std::unordered_map<Key, int32_t, Hash> local;
        for (int64_t r = lo; r < hi && local.size() <= 256; ++r) local.emplace(key_at(r), 0);
        std::lock_guard<std::mutex> lk(mu);
        for (const auto &kv : local) table.emplace(kv.first, 0);
        if (local.size() > 256 || table.size() > 256) overflow = true;
    }, 1 << 16);
    if (overflow || table.size() > 256) return false;
    std::vector<Key> keys;
    for (const auto &kv : table) keys.push_back(kv.first);
    std::sort(keys.begin(), keys.end(), [](const Key &a, const Key &b) { return std::memcmp(a.b, b.b, K) < 0; });
    for (size_t q = 0; q < keys.size(); ++q) table[keys[q]] = (int32_t)q;
    parallel_for(ns, [&](int64_t lo, int64_t hi) {
        for (int64_t r = lo; r < hi; ++r)
            c->h_rec_id2[r].x = (int32_t)((uint32_t)c->h_rec_id2[r].x | ((uint32_t)table.at(key_at(r)) << 22));
    }, 1 << 16);
    c->n_tab = (int64_t)keys.size();
    c->h_rec_a.assign(keys.size() * K, 0);
    for (size_t q = 0; q < keys.size(); ++q) std::memcpy(c->h_rec_a.data() + q * K, keys[q].b, K);
    group_table_records<R>(c);
    return true;
}

// weak constraints held by this context (owned first): distinct nodes with combined weights w0_j - w1_j;
// per owned free vertex the list of (constraint, w0_i - w1_i) in input order.  Also the fast path of
// pbng_update_constraints (colouring unchanged: only these arrays are rebuilt and uploaded).
template <class R>
void build_constraint_arrays(pbng_ctx *c) {
    const size_t s = sizeof(R), s4 = 4 * sizeof(R);
    const int64_t ncl = (int64_t)c->cons_local.size();
    const int64_t ncap = std::max<int64_t>(ncl, 1);
    c->h_c_n.assign((size_t)ncap, 0);
    c->h_c_node.assign((size_t)ncap * kWcMaxNodes, 0);
    c->h_c_w.assign((size_t)ncap * kWcMaxNodes * s, 0);
    c->h_c_anchor.assign((size_t)ncap * s4, 0);
    c->h_c_K.assign((size_t)ncap * kWcMaxNodes * s, 0);
    std::vector<std::pair<int32_t, int32_t>> by_gid;  // (global id, local id), ascending global id
    for (int64_t li = 0; li < ncl; ++li) by_gid.push_back({c->cons_local[li], (int32_t)li});
    std::sort(by_gid.begin(), by_gid.end());
    std::vector<std::vector<std::pair<int32_t, double>>> per_v((size_t)c->n_free);
    for (const auto &gl : by_gid) {
        const int32_t li = gl.second;
        const pbng_weak_constraint &w = c->wc[gl.first];
        int32_t nodes[kWcMaxNodes];
        double wt[kWcMaxNodes];
        int nn = 0;
        auto add = [&](int32_t node, double weight) {
            for (int q = 0; q < nn; ++q)
                if (nodes[q] == node) { wt[q] += weight; return; }
            nodes[nn] = node;
            wt[nn] = weight;
            ++nn;
        };
        for (int q = 0; q < w.n0; ++q) add(w.idx0[q], w.w0[q]);
        for (int q = 0; q < w.n1; ++q) add(w.idx1[q], -w.w1[q]);
        c->h_c_n[li] = nn;
        for (int q = 0; q < nn; ++q) {
            const int32_t vi = c->orig2int[nodes[q]];
            c->h_c_node[kWcMaxNodes * li + q] = vi;
            put1<R>(c->h_c_w, kWcMaxNodes * li + q, wt[q]);
            if (vi >= 0 && vi < c->n_free) per_v[vi].push_back({li, wt[q]});
        }
        if (w.n1 == 0) put4<R>(c->h_c_anchor, li, w.anchor[0], w.anchor[1], w.anchor[2], 0.0);
        for (int q = 0; q < 6; ++q) put1<R>(c->h_c_K, kWcMaxNodes * li + q, w.K[q]);
    }
    c->h_wc_off.assign((size_t)c->n_free + 1, 0);
    for (int64_t i = 0; i < c->n_free; ++i) c->h_wc_off[i + 1] = c->h_wc_off[i] + (int32_t)per_v[i].size();
    c->n_vc = c->h_wc_off[c->n_free];
    c->h_wc_cid.assign((size_t)std::max<int64_t>(c->n_vc, 1), 0);
    c->h_wc_d.assign((size_t)std::max<int64_t>(c->n_vc, 1) * s, 0);
    for (int64_t i = 0; i < c->n_free; ++i)
        for (size_t q = 0; q < per_v[i].size(); ++q) {
            c->h_wc_cid[c->h_wc_off[i] + q] = per_v[i][q].first;
            put1<R>(c->h_wc_d, c->h_wc_off[i] + q, per_v[i][q].second);
        }

}

template <class R>
void build_layout(pbng_ctx *c, const std::vector<int64_t> &vt_off, const std::vector<int32_t> &vt) {
    const int64_t nv = c->nv, nb = c->nb;
    const size_t s = sizeof(R), s4 = 4 * sizeof(R);
    const double cmu = 1.0 / (2.0 * (1.0 + c->nu));
    const double clam = c->nu / ((1.0 + c->nu) * (1.0 - 2.0 * c->nu));
    auto Ee = [&](int64_t e) { return c->E.size() == 1 ? c->E[0] : c->E[(size_t)e]; };

    // chunks and degrees (path-ordered NH records: records per vertex incl. load-only ones)
    c->path_rec = use_path_records(c);
    c->rest_rec = use_rest_records(c);
    c->col_chunk.assign(c->ncol + 1, 0);
    c->h_deg.assign(c->n_free, 0);
    auto vertex_link = [&](int32_t o, std::vector<std::array<int32_t, 3>> &link) {  // other vertices per incident tet
        link.clear();
        for (int64_t q = vt_off[o]; q < vt_off[o + 1]; ++q) {
            const int32_t *t = c->tets.data() + 4 * vt[q];
            std::array<int32_t, 3> tr;
            int m = 0;
            for (int sl = 0; sl < 4; ++sl)
                if (t[sl] != o) tr[m++] = t[sl];
            link.push_back(tr);
        }
    };
    if (c->path_rec) c->h_path0.assign((size_t)std::max<int64_t>(c->n_free, 1), make_int2(0, 0));
    parallel_for(c->n_free, [&](int64_t lo, int64_t hi) {
        std::vector<std::array<int32_t, 3>> link;
        std::vector<PathRec> prec;
        PathMemo memo;
        for (int64_t i = lo; i < hi; ++i) {
            const int32_t o = c->int2orig[i];
            if (c->path_rec) {
                vertex_link(o, link);
                int32_t p0[2];
                vertex_path_records(link, (uint32_t)o, prec, p0, &memo);
                c->h_deg[i] = (int32_t)prec.size();
                c->h_path0[i] = prec.empty() ? make_int2((int32_t)i, (int32_t)i)
                                             : make_int2(c->orig2int[p0[0]], c->orig2int[p0[1]]);
            } else {
                c->h_deg[i] = (int32_t)(vt_off[o + 1] - vt_off[o]);
            }
        }
    }, 1024);
    c->h_chunk_off.clear();
    c->h_chunk_v.clear();
    c->h_chunk_off.push_back(0);
    int64_t n_chunks = 0;
    c->col_chunk_mid.assign(c->ncol, 0);
    if (c->col_nsend.size() != (size_t)c->ncol) c->col_nsend.assign(c->ncol, 0);
    for (int32_t col = 0; col < c->ncol; ++col) {
        c->col_chunk[col] = n_chunks;
        // two parts, each chunked from its own start: the halo-send vertices, then the rest
        for (int part = 0; part < 2; ++part) {
            if (part == 1) c->col_chunk_mid[col] = n_chunks;
            const int32_t ns = c->col_nsend[col];
            const int32_t v0 = c->col_vbegin[col] + (part ? ns : 0), nc = part ? c->col_nfree[col] - ns : ns;
            for (int32_t k = 0; k < nc; k += kChunk) {
                const int32_t cnt = std::min<int32_t>(kChunk, nc - k);
                int32_t width = 0;
                for (int32_t q = 0; q < cnt; ++q) width = std::max(width, c->h_deg[v0 + k + q]);
                c->h_chunk_v.push_back(make_int2(v0 + k, cnt));
                c->h_chunk_off.push_back(c->h_chunk_off.back() + (int64_t)width * kChunk);
                ++n_chunks;
            }
        }
    }
    c->col_chunk[c->ncol] = n_chunks;
    c->n_chunks = n_chunks;
    c->n_slots = c->h_chunk_off.back();
    c->n_pairs = 0;
    c->n_records = 0;
    for (int64_t i = 0; i < c->n_free; ++i) {
        const int32_t o = c->int2orig[i];
        c->n_pairs += vt_off[o + 1] - vt_off[o];
        c->n_records += c->h_deg[i];
    }

    // pair records
    const int64_t ns = std::max<int64_t>(c->n_slots, 1);
    c->h_rec_id.assign(c->path_rec ? 1 : (size_t)ns, make_int4(0, 0, 0, 0));
    c->h_rec_id2.assign(c->path_rec ? (size_t)ns : 1, make_int2(0, 0));
    c->h_rec_a.assign(c->rest_rec ? s4 : (size_t)ns * s4, 0);  // rest-recompute records: unused
    const bool nh = c->model == MODEL_NH;
    // NH: unused, except the batched sh-6 path records' precomputed material scalars {V mu, V lambda,
    // V (mu + lambda), 2 V mu |g_i|^2} (pbng_kernels.cu contrib_nh2v)
    const bool b2v = nh && c->path_rec && layout_lane_shift(c) == 6;
    c->h_rec_b.assign(nh && !b2v ? s4 : (size_t)ns * s4, 0);
    // rec_c: FCR g3z (+ VE in fp64); NH: VE in fp64, unused in fp32 (VE rides in rec_id.w)
    // rest-recompute records: rec_c holds E_e/6 in fp64 (fp32: in rec_id.y)
    const size_t rec_c_bytes = nh ? (c->dtype == DT_F64 ? s : 0) : (c->dtype == DT_F64 ? 2 * s : s);
    c->h_rest.assign(c->rest_rec ? (size_t)std::max<int64_t>(c->n_local, 1) * s4 : 0, 0);
    if (c->rest_rec)
        for (int64_t i = 0; i < c->n_local; ++i) {
            const double *X = c->X.data() + 3 * (size_t)c->int2orig[i];
            put4<R>(c->h_rest, i, X[0], X[1], X[2], 0.0);
        }
    c->h_rec_c.assign(std::max<size_t>((size_t)ns * rec_c_bytes, s), 0);
    parallel_for(n_chunks, [&](int64_t ch_lo, int64_t ch_hi) {  // chunks write disjoint record slots
    std::vector<std::array<int32_t, 3>> link;
    std::vector<PathRec> prec;
    PathMemo memo;
    for (int64_t ch = ch_lo; ch < ch_hi; ++ch) {
        const int2 cv = c->h_chunk_v[ch];
        for (int32_t lane = 0; lane < cv.y; ++lane) {
            const int32_t vi = cv.x + lane, o = c->int2orig[vi];
            if (c->path_rec) {
                // path-ordered records: slot order (S0, S1, S2) after the push; s'_k and det B' follow the
                // slots (det B' = sgn(pi) det B keeps J and cof(F) g_i, pbng_kernels.cu "path records")
                vertex_link(o, link);
                int32_t p0[2];
                vertex_path_records(link, (uint32_t)o, prec, p0, &memo);
                for (size_t k = 0; k < prec.size(); ++k) {
                    const PathRec &pr = prec[k];
                    const int64_t r = c->h_chunk_off[ch] + (int64_t)k * kChunk + lane;
                    const int32_t code = c->orig2int[pr.vnew] | (pr.drop << 30);
                    if (pr.tet < 0) {  // load-only: VE = 0 and zero rest data contribute exactly 0
                        c->h_rec_id2[r] = make_int2(code, 0);
                        if (!c->rest_rec) put4<R>(c->h_rec_a, r, 0.0, 0.0, 0.0, 0.0);
                        if (c->dtype == DT_F64) put1<R>(c->h_rec_c, r, 0.0);
                        continue;
                    }
                    const int64_t e = vt[vt_off[o] + pr.tet];
                    if (c->rest_rec) {  // E_e / 6: V_e E_e = |det Dm'| E_e / 6 with Dm' rebuilt in slot order
                        const double E6 = Ee(e) / 6.0;
                        int2 id = make_int2(code, 0);
                        if (c->dtype == DT_F32) {
                            const float ef = (float)E6;
                            std::memcpy(&id.y, &ef, 4);
                        } else {
                            put1<R>(c->h_rec_c, r, E6);
                        }
                        c->h_rec_id2[r] = id;
                        continue;
                    }
                    const int32_t *t = c->tets.data() + 4 * e;
                    int a = 0;
                    while (t[a] != o) ++a;
                    int32_t oid[3];
                    double g[3][3], gi[3], sj[3];
                    int m = 0;
                    for (int sl = 0; sl < 4; ++sl) {
                        if (sl == a) continue;
                        oid[m] = t[sl];
                        shape_grad(c, e, sl, g[m]);
                        ++m;
                    }
                    shape_grad(c, e, a, gi);
                    for (int q2 = 0; q2 < 3; ++q2) sj[q2] = g[q2][0] * gi[0] + g[q2][1] * gi[1] + g[q2][2] * gi[2];
                    const double Bp[9] = {g[0][0], g[0][1], g[0][2], g[1][0], g[1][1], g[1][2], g[2][0], g[2][1], g[2][2]};
                    int pi[3];
                    for (int k2 = 0; k2 < 3; ++k2) {
                        pi[k2] = 0;
                        while (oid[pi[k2]] != pr.slot[k2]) ++pi[k2];
                    }
                    const int inv = (pi[0] > pi[1]) + (pi[0] > pi[2]) + (pi[1] > pi[2]);
                    const double sgn = (inv & 1) ? -1.0 : 1.0;
                    const double VE = c->V[e] * Ee(e);
                    int2 id = make_int2(code, 0);
                    if (c->dtype == DT_F32) {
                        const float vf = (float)VE;
                        std::memcpy(&id.y, &vf, 4);
                    }
                    c->h_rec_id2[r] = id;
                    put4<R>(c->h_rec_a, r, sj[pi[0]], sj[pi[1]], sj[pi[2]], sgn * det3(Bp));
                    if (b2v) {
                        const double Vmu = VE * cmu, Vlam = VE * clam;
                        put4<R>(c->h_rec_b, r, Vmu, Vlam, Vmu + Vlam, -2.0 * Vmu * (sj[0] + sj[1] + sj[2]));
                    }
                    if (c->dtype == DT_F64) put1<R>(c->h_rec_c, r, VE);
                }
                continue;
            }
            int k = 0;
            for (int64_t q = vt_off[o]; q < vt_off[o + 1]; ++q, ++k) {
                const int64_t e = vt[q];
                const int32_t *t = c->tets.data() + 4 * e;
                int a = 0;
                while (t[a] != o) ++a;
                int ids[3], m = 0;
                double g[3][3];
                for (int sl = 0; sl < 4; ++sl) {
                    if (sl == a) continue;
                    ids[m] = c->orig2int[t[sl]];
                    shape_grad(c, e, sl, g[m]);
                    ++m;
                }
                const int64_t r = c->h_chunk_off[ch] + (int64_t)k * kChunk + lane;
                const double VE = c->V[e] * Ee(e);
                int4 id = make_int4(ids[0], ids[1], ids[2], 0);
                if (c->dtype == DT_F32) {
                    const float vf = (float)VE;
                    std::memcpy(&id.w, &vf, 4);
                }
                c->h_rec_id[r] = id;
                if (nh) {
                    // compact Neo-Hookean record: s_j = g_j . g_i and det B, with B = rows g_j of the three
                    // other vertices (pbng_kernels.cu, Pair<R, MODEL_NH>); |g_i|^2 = -(s_1 + s_2 + s_3)
                    double gi[3], sj[3];
                    shape_grad(c, e, a, gi);
                    const double Bp[9] = {g[0][0], g[0][1], g[0][2], g[1][0], g[1][1], g[1][2], g[2][0], g[2][1], g[2][2]};
                    for (int q2 = 0; q2 < 3; ++q2) sj[q2] = g[q2][0] * gi[0] + g[q2][1] * gi[1] + g[q2][2] * gi[2];
                    put4<R>(c->h_rec_a, r, sj[0], sj[1], sj[2], det3(Bp));
                    if (c->dtype == DT_F64) put1<R>(c->h_rec_c, r, VE);
                } else {
                    put4<R>(c->h_rec_a, r, g[0][0], g[0][1], g[0][2], g[1][0]);
                    put4<R>(c->h_rec_b, r, g[1][1], g[1][2], g[2][0], g[2][1]);
                    if (c->dtype == DT_F64) {
                        put1<R>(c->h_rec_c, 2 * r, g[2][2]);
                        put1<R>(c->h_rec_c, 2 * r + 1, VE);
                    } else {
                        put1<R>(c->h_rec_c, r, g[2][2]);
                    }
                }
            }
        }
    }

    }, 64);
    c->tab_rec = false;
    c->n_tab = 0;
    if (!c->rest_rec && want_table_records(c)) c->tab_rec = build_rest_table<R>(c);

    // body force f^ext_i = sum_e R^0 g V_e / 4, free vertices
    const bool has_fext = c->density > 0 && (c->grav[0] != 0 || c->grav[1] != 0 || c->grav[2] != 0);
    c->h_fext.assign(has_fext ? (size_t)std::max<int64_t>(c->n_free, 1) * s4 : 0, 0);
    if (has_fext)
        for (int64_t i = 0; i < c->n_free; ++i) {
            const int32_t o = c->int2orig[i];
            double m = 0;
            for (int64_t q = vt_off[o]; q < vt_off[o + 1]; ++q) m += c->density * c->V[vt[q]] / 4.0;
            put4<R>(c->h_fext, i, m * c->grav[0], m * c->grav[1], m * c->grav[2], 0.0);
        }

    // lumped masses m_ii = int R^0 N_i dX = sum_e R^0 V_e / 4, owned free vertices
    c->h_mass.assign((size_t)std::max<int64_t>(c->n_free, 1) * s, 0);
    for (int64_t i = 0; i < c->n_free; ++i) {
        const int32_t o = c->int2orig[i];
        double m = 0;
        for (int64_t q = vt_off[o]; q < vt_off[o + 1]; ++q) m += c->density * c->V[vt[q]] / 4.0;
        put1<R>(c->h_mass, i, m);
    }

    build_constraint_arrays<R>(c);

    // tet records for the energy pass (the tets this context owns)
    const int64_t ntl = (int64_t)c->tet_local.size();
    const int64_t ntr = std::max<int64_t>(ntl, 1);
    c->h_tet_id.assign((size_t)ntr, make_int4(0, 0, 0, 0));
    c->h_tet_a.assign((size_t)ntr * s4, 0);
    c->h_tet_b.assign((size_t)ntr * s4, 0);
    c->h_tet_c.assign((size_t)ntr * s4, 0);
    for (int64_t q = 0; q < ntl; ++q) {
        const int64_t e = c->tet_local[q];
        const int32_t *t = c->tets.data() + 4 * e;
        const double *B = c->Bm.data() + 9 * e;
        c->h_tet_id[q] = make_int4(c->orig2int[t[0]], c->orig2int[t[1]], c->orig2int[t[2]], c->orig2int[t[3]]);
        put4<R>(c->h_tet_a, q, B[0], B[1], B[2], B[3]);
        put4<R>(c->h_tet_b, q, B[4], B[5], B[6], B[7]);
        put4<R>(c->h_tet_c, q, B[8], c->V[e] * Ee(e), c->V[e], 0.0);
    }

    // Dirichlet targets of the held pinned vertices as Real4 [nb][n_pinned_local]
    const int64_t np = (int64_t)c->pinned.size(), npl = (int64_t)c->local_pinned.size();
    c->h_targets.assign((size_t)std::max<int64_t>(nb * npl, 1) * s4, 0);
    for (int64_t b = 0; b < nb; ++b)
        for (int64_t k = 0; k < npl; ++k) {
            const double *t = c->targets.data() + 3 * (b * np + c->local_pinned[k]);
            put4<R>(c->h_targets, b * npl + k, t[0], t[1], t[2], 0.0);
        }

    // problem constants
    Problem &p = c->prob;
    p.dtype = c->dtype;
    p.model = c->model;
    p.n_vertices = c->n_local;
    p.n_global = nv;
    p.n_free = c->n_local_free;
    p.n_pinned = npl;
    p.n_tets = ntl;
    p.n_cons = c->n_cons_owned;
    p.n_chunks = n_chunks;
    p.n_batch = c->nb;
    p.x_stride = (int64_t)align_up((size_t)std::max<int64_t>(c->n_local, 1), 64);
    // batched layouts: fp32 Neo-Hookean -> the component-interleaved two-sample layout of
    // sweep_batched2_kernel (sh 6), otherwise sample-minor groups of 32 (sh 5)
    p.lane_shift = layout_lane_shift(c);
    p.path = c->path_rec;
    p.path_mode = !c->path_rec ? 0 : c->rest_rec ? 2 : c->tab_rec ? 3 : 1;
    p.cmu = cmu;
    p.clam = clam;
    for (int k = 0; k < 3; ++k) p.rho_g[k] = c->density * c->grav[k];
    p.has_fext = has_fext;
    p.has_wc = c->n_vc > 0;
    p.n_own = c->n_free;
    p.inv_dt2 = 0.0;
    const int64_t items = ntl + c->n_cons_owned + c->n_free;
    p.ge = (int)std::max<int64_t>(1, std::min<int64_t>((items + kRedBlock - 1) / kRedBlock, 1184));
    p.gr = (int)std::max<int64_t>(1, std::min<int64_t>((n_chunks * kChunk + kRedBlock - 1) / kRedBlock, 1184));
}

// Pipelined schedule (pbng_kernels.cu sweep_pipe_kernel): for every chunk, the chunks holding the other
// nodes of its vertices' stencils (tets and weak constraints) and the chunk itself, each tagged with
// whether it belongs to an earlier colour (must have finished the current iteration) or not (the
// previous one).  Only for an undecomposed context (ghost values arrive by halo exchange between
// colour passes, which needs the per-colour launches).
void build_pipeline(pbng_ctx *c, const std::vector<int64_t> &vt_off, const std::vector<int32_t> &vt) {
    c->h_dep_off.assign((size_t)c->n_chunks + 1, 0);
    c->h_deps.clear();
    if (c->n_ranks > 1) return;  // the pipelined schedule is unavailable (pipeline_available)
    std::vector<int32_t> chunk_of((size_t)std::max<int64_t>(c->n_free, 1), -1), chunk_col((size_t)std::max<int64_t>(c->n_chunks, 1), 0);
    for (int32_t col = 0; col < c->ncol; ++col)
        for (int64_t ch = c->col_chunk[col]; ch < c->col_chunk[col + 1]; ++ch) {
            chunk_col[ch] = col;
            const int2 cv = c->h_chunk_v[ch];
            for (int32_t q = 0; q < cv.y; ++q) chunk_of[cv.x + q] = (int32_t)ch;
        }
    // per chunk in parallel (each thread its own "already listed" stamps), then concatenated in chunk order
    std::vector<std::vector<int32_t>> lists((size_t)c->n_chunks);
    parallel_for(c->n_chunks, [&](int64_t lo, int64_t hi) {
        std::vector<int64_t> stamp((size_t)std::max<int64_t>(c->n_chunks, 1), -1);  // chunk already listed for ch
        for (int64_t ch = lo; ch < hi; ++ch) {
            std::vector<int32_t> &tmp = lists[ch];
            tmp.push_back((int32_t)ch);
            stamp[ch] = ch;
            const int2 cv = c->h_chunk_v[ch];
            auto add = [&](int32_t j) {
                if (j >= 0 && j < c->n_free && stamp[chunk_of[j]] != ch) {
                    stamp[chunk_of[j]] = ch;
                    tmp.push_back(chunk_of[j]);
                }
            };
            for (int32_t q = 0; q < cv.y; ++q) {
                const int32_t i = cv.x + q, o = c->int2orig[i];
                for (int64_t k = vt_off[o]; k < vt_off[o + 1]; ++k) {
                    const int32_t *t = c->tets.data() + 4 * vt[k];
                    for (int a = 0; a < 4; ++a) add(c->orig2int[t[a]]);
                }
                for (int32_t k = c->h_wc_off[i]; k < c->h_wc_off[i + 1]; ++k) {
                    const int32_t cid = c->h_wc_cid[k];
                    for (int32_t m = 0; m < c->h_c_n[cid]; ++m) add(c->h_c_node[kWcMaxNodes * cid + m]);
                }
            }
            std::sort(tmp.begin(), tmp.end());
        }
    }, 64);
    for (int64_t ch = 0; ch < c->n_chunks; ++ch) {
        for (int32_t y : lists[ch]) c->h_deps.push_back((y << 1) | (chunk_col[y] < chunk_col[ch] ? 1 : 0));
        c->h_dep_off[ch + 1] = (int32_t)c->h_deps.size();
    }
}

// Boundary triangles of the mesh (faces of exactly one tet) in order of (tet, local face k), face k = the
// other three vertices in ascending local order, the last two swapped when the rest-state normal
// (v1 - v0) x (v2 - v0) points towards local vertex k (include/pbng.h pbng_detect_contacts), and bodies
// = connected components of tets sharing a vertex, labelled by their smallest vertex index.  Only for
// an undecomposed context.
void surface_original(pbng_ctx *c);
void build_surface(pbng_ctx *c) {
    c->h_surf.clear();
    c->h_sv.clear();
    c->prob.n_surf = c->prob.n_sv = 0;
    c->prob.n_cbuckets = 1;
    if (c->n_ranks > 1 || c->nt == 0) return;
#ifdef PBNG_NO_SURF_CACHE
    c->surf_cached = false;
#endif
    if (!c->surf_cached) surface_original(c);  // mesh-only: computed once, re-laid out by id mapping
    const size_t nf = c->surf_orig.size() / 3;
    for (size_t f = 0; f < nf; ++f) {
        const int32_t *v = &c->surf_orig[3 * f];
        c->h_surf.push_back(make_int4(c->orig2int[v[0]], c->orig2int[v[1]], c->orig2int[v[2]], c->surf_body[f]));
    }
    std::vector<char> is_pinned((size_t)c->nv, 0);
    for (int32_t p : c->pinned) is_pinned[p] = 1;
    for (size_t k = 0; k < c->surf_verts.size(); ++k) {
        const int32_t v = c->surf_verts[k];
        if (!is_pinned[v]) c->h_sv.push_back(make_int2(c->orig2int[v], c->surf_vbody[k]));
    }
    c->prob.n_surf = (int64_t)c->h_surf.size();
    c->prob.n_sv = (int64_t)c->h_sv.size();
    int64_t nb = 1;
    while (nb < 16 * std::max<int64_t>(c->prob.n_surf, 1)) nb <<= 1;
    c->prob.n_cbuckets = nb;
}

// the boundary of the rest mesh in original ids (surf_orig, surf_body, surf_verts, surf_vbody)
void surface_original(pbng_ctx *c) {
    c->surf_orig.clear();
    c->surf_body.clear();
    c->surf_verts.clear();
    c->surf_vbody.clear();
    const int64_t nt = c->nt, nv = c->nv;
    // union-find over vertices
    std::vector<int32_t> par((size_t)nv);
    for (int64_t v = 0; v < nv; ++v) par[v] = (int32_t)v;
    auto root = [&](int32_t v) {
        while (par[v] != v) { par[v] = par[par[v]]; v = par[v]; }
        return v;
    };
    for (int64_t e = 0; e < nt; ++e)
        for (int a = 1; a < 4; ++a) {
            const int32_t r0 = root(c->tets[4 * e]), r1 = root(c->tets[4 * e + a]);
            if (r0 != r1) par[std::max(r0, r1)] = std::min(r0, r1);
        }
    std::vector<int32_t> body((size_t)nv);
    for (int64_t v = 0; v < nv; ++v) body[v] = root((int32_t)v);  // the component's minimum vertex
    // a face is on the boundary iff no other tet has the same vertex triple: faces are bucketed by their
    // smallest vertex (CSR), and each bucket's few faces are matched on the other two (sorted) vertices
    auto face_key = [&](int64_t e, int f, int32_t k[3]) {
        int m = 0;
        for (int a = 0; a < 4; ++a)
            if (a != f) k[m++] = c->tets[4 * e + a];
        std::sort(k, k + 3);
    };
    std::vector<int64_t> off((size_t)nv + 1, 0);
    for (int64_t e = 0; e < nt; ++e)
        for (int f = 0; f < 4; ++f) {
            int32_t k[3];
            face_key(e, f, k);
            off[k[0] + 1]++;
        }
    for (int64_t v = 0; v < nv; ++v) off[v + 1] += off[v];
    std::vector<int64_t> fid((size_t)(4 * nt)), fill(off.begin(), off.end() - 1);
    for (int64_t e = 0; e < nt; ++e)
        for (int f = 0; f < 4; ++f) {
            int32_t k[3];
            face_key(e, f, k);
            fid[fill[k[0]]++] = 4 * e + f;
        }
    std::vector<char> boundary((size_t)(4 * nt), 0);
    parallel_for(nv, [&](int64_t lo, int64_t hi) {
        std::vector<std::pair<uint64_t, int64_t>> b;
        for (int64_t v = lo; v < hi; ++v) {
            b.clear();
            for (int64_t q = off[v]; q < off[v + 1]; ++q) {
                int32_t k[3];
                face_key(fid[q] / 4, (int)(fid[q] % 4), k);
                b.push_back({(uint64_t)(uint32_t)k[1] << 32 | (uint32_t)k[2], fid[q]});
            }
            std::sort(b.begin(), b.end());
            for (size_t i = 0; i < b.size();) {
                size_t j = i + 1;
                while (j < b.size() && b[j].first == b[i].first) ++j;
                if (j == i + 1) boundary[b[i].second] = 1;
                i = j;
            }
        }
    });
    std::vector<char> on_surf((size_t)nv, 0);
    for (int64_t e = 0; e < nt; ++e)
        for (int f = 0; f < 4; ++f) {
            if (!boundary[4 * e + f]) continue;
            int32_t v[3];
            int m = 0;
            for (int a = 0; a < 4; ++a)
                if (a != f) v[m++] = c->tets[4 * e + a];
            const double *x0 = &c->X[3 * v[0]], *x1 = &c->X[3 * v[1]], *x2 = &c->X[3 * v[2]],
                         *xk = &c->X[3 * c->tets[4 * e + f]];
            const double u[3] = {x1[0] - x0[0], x1[1] - x0[1], x1[2] - x0[2]};
            const double w[3] = {x2[0] - x0[0], x2[1] - x0[1], x2[2] - x0[2]};
            const double n[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
            if (n[0] * (xk[0] - x0[0]) + n[1] * (xk[1] - x0[1]) + n[2] * (xk[2] - x0[2]) > 0.0) std::swap(v[1], v[2]);
            for (int a = 0; a < 3; ++a) {
                c->surf_orig.push_back(v[a]);
                on_surf[v[a]] = 1;
            }
            c->surf_body.push_back(body[v[0]]);
        }
    for (int64_t v = 0; v < nv; ++v)
        if (on_surf[v]) {
            c->surf_verts.push_back((int32_t)v);
            c->surf_vbody.push_back(body[v]);
        }
    c->surf_cached = true;
}

// Incremental recolouring of pbng_update_constraints: the nodes incident to the new
// constraints (nodes_new) are visited in ascending index; each keeps its colour unless a node sharing a
// stencil (tet or constraint of the new set) holds it, in which case it takes the least colour no such
// node holds (reading Z20).  `nodes` = distinct node lists of the new constraint set.
std::vector<int32_t> recolour_incremental(const pbng_ctx *c, const std::vector<std::vector<int32_t>> &nodes,
                                          const std::vector<char> &is_new, int64_t *changed) {
    const int64_t nv = c->nv, nt = c->nt;
    std::vector<int32_t> col = c->colour;
    std::vector<std::vector<int32_t>> vcons((size_t)nv);  // vertex -> constraints
    std::vector<char> extra((size_t)nv, 0);
    for (size_t q = 0; q < nodes.size(); ++q)
        for (int32_t v : nodes[q]) {
            vcons[v].push_back((int32_t)q);
            if (is_new[q]) extra[v] = 1;
        }
    std::vector<std::vector<int32_t>> vtets((size_t)nv);
    if (!c->inc_off.empty()) {  // the cached incidence (ascending tet index, as the scan below)
        for (int64_t v = 0; v < nv; ++v)
            if (extra[v]) vtets[v].assign(c->inc.begin() + c->inc_off[v], c->inc.begin() + c->inc_off[v + 1]);
    } else {
        for (int64_t e = 0; e < nt; ++e)
            for (int a = 0; a < 4; ++a)
                if (extra[c->tets[4 * e + a]]) vtets[c->tets[4 * e + a]].push_back((int32_t)e);
    }
    int32_t ncol = 0;
    for (int32_t k : col) ncol = std::max(ncol, k + 1);
    *changed = 0;
    std::vector<char> used;
    for (int64_t v = 0; v < nv; ++v) {
        if (!extra[v]) continue;
        used.assign((size_t)ncol + 1, 0);
        for (int32_t e : vtets[v])
            for (int a = 0; a < 4; ++a)
                if (c->tets[4 * e + a] != v) used[col[c->tets[4 * e + a]]] = 1;
        for (int32_t q : vcons[v])
            for (int32_t u : nodes[q])
                if (u != v) used[col[u]] = 1;
        if (!used[col[v]]) continue;
        int32_t k = 0;
        while (used[k]) ++k;
        col[v] = k;
        ncol = std::max(ncol, k + 1);
        ++*changed;
    }
    return col;
}

pbng_status validate_wc(const pbng_ctx *c, const pbng_weak_constraint *wc, int64_t n_wc, const char *who) {
    const std::string w0(who);
    for (int64_t q = 0; q < n_wc; ++q) {
        const pbng_weak_constraint &w = wc[q];
        if (w.n0 < 1 || w.n0 > 4 || w.n1 < 0 || w.n1 > 4)
            return fail(PBNG_E_INVALID_ARGUMENT, w0 + ": weak constraint " + std::to_string(q) + " has bad node counts");
        for (int a = 0; a < w.n0; ++a)
            if (w.idx0[a] < 0 || w.idx0[a] >= c->nv || !std::isfinite(w.w0[a]))
                return fail(PBNG_E_INDEX_OUT_OF_RANGE, w0 + ": weak constraint " + std::to_string(q) + " side 0");
        for (int a = 0; a < w.n1; ++a)
            if (w.idx1[a] < 0 || w.idx1[a] >= c->nv || !std::isfinite(w.w1[a]))
                return fail(PBNG_E_INDEX_OUT_OF_RANGE, w0 + ": weak constraint " + std::to_string(q) + " side 1");
        for (int a = 0; a < 6; ++a)
            if (!std::isfinite(w.K[a])) return fail(PBNG_E_INVALID_ARGUMENT, w0 + ": non-finite K");
        for (int a = 0; a < 3; ++a)
            if (!std::isfinite(w.anchor[a])) return fail(PBNG_E_INVALID_ARGUMENT, w0 + ": non-finite anchor");
    }
    return PBNG_OK;
}

std::vector<int32_t> distinct_nodes(const pbng_weak_constraint &w) {
    std::vector<int32_t> n;
    for (int a = 0; a < w.n0; ++a) n.push_back(w.idx0[a]);
    for (int a = 0; a < w.n1; ++a) n.push_back(w.idx1[a]);
    std::sort(n.begin(), n.end());
    n.erase(std::unique(n.begin(), n.end()), n.end());
    return n;
}

bool pipeline_available(const pbng_ctx *c) {
    // path-ordered records are walked by one warp per chunk: the pipelined kernel then runs one-warp items
    return c->n_ranks == 1 && c->prob.lane_shift == 0 && c->n_chunks > 0 && (!c->path_rec || problem_split(c) == 1);
}

int problem_split(const pbng_ctx *c);

// schedule pbng_iterate uses: 1 = one launch per colour pass, 2 = pipelined (PBNG_SCHEDULE env overrides
// auto).  Auto pipelines small problems, whose colour passes are too short to fill the machine (launch
// and barrier latency dominate; measured 1.3x on config 1, 1.03x on config 2); large ones keep the colour
// launches, whose neighbour gathers may use the read-only L1 path (the pipelined kernel needs coherent
// loads, measured 7% slower on config 3 and 15% on config 5).
int effective_schedule(const pbng_ctx *c) {
    static const int env = [] {
        const char *e = getenv("PBNG_SCHEDULE");
        return e ? atoi(e) : 0;
    }();
    int want = c->schedule != 0 ? c->schedule : env;
    if (want == 0) {  // fewer 32-vertex chunks per colour than 8 per SM: the colour passes cannot fill the GPU
        int64_t gfree = 0;
        for (int64_t k : c->gcol_nfree) gfree += k;
        const int64_t chunks_per_colour = gfree * c->nb / kChunk / std::max(c->ncol, 1);
        want = chunks_per_colour < 148 * 8 ? 2 : 1;
    }
    return (want == 2 && pipeline_available(c)) ? 2 : 1;
}

void plan_workspace(pbng_ctx *c) {
    size_t off = 0;
    auto take = [&](Region &r, size_t bytes) {
        r.off = off;
        r.bytes = std::max<size_t>(bytes, 1);
        off = align_up(off + r.bytes, 256);
    };
    const Problem &p = c->prob;
    const size_t s = c->real_size(), s4 = c->real4_size();
    // position buffers and staging first: their offsets depend only on (n_batch, vertices held, dtype,
    // layout shift), so a re-layout with the same vertex set (pbng_update_constraints) leaves them in place
    // and the iterate can be carried over on the device
    {
        size_t groups = (size_t)((c->nb + (1 << p.lane_shift) - 1) >> p.lane_shift);
        if (p.lane_shift == 5) groups += groups & 1;
        for (int k = 0; k < 3; ++k) take(c->r_x[k], (groups << p.lane_shift) * (size_t)p.x_stride * s4);
        take(c->r_xt, (groups << p.lane_shift) * (size_t)p.x_stride * s4);
        take(c->r_stage, (size_t)c->nb * (size_t)c->nv * 3 * s);
        take(c->r_stage2, (size_t)c->nb * (size_t)c->nv * 3 * s);
    }
    const int64_t ns = std::max<int64_t>(c->n_slots, 1);
    take(c->r_rec_id, (size_t)ns * (c->path_rec ? 8 : 16));
    take(c->r_path0, c->h_path0.size() * 8);
    take(c->r_rec_a, c->h_rec_a.size());
    take(c->r_rest, c->h_rest.size());
    take(c->r_rec_b, c->h_rec_b.size());
    take(c->r_rec_c, c->h_rec_c.size());
    take(c->r_chunk_off, c->h_chunk_off.size() * 8);
    take(c->r_chunk_v, std::max<size_t>(c->h_chunk_v.size(), 1) * 8);
    take(c->r_deg, std::max<size_t>(c->h_deg.size(), 1) * 4);
    take(c->r_fext, c->h_fext.size());
    // weak constraints get headroom (pbng_update_constraints' fast path rewrites them in place): room for
    // a contact at every free boundary vertex (up to 4 free nodes each) on top of twice the current set
    const size_t ncl = c->h_c_n.size(), nvc = c->h_wc_cid.size();
    c->wc_cap = std::max<size_t>(2 * ncl, ncl + c->h_sv.size() + 64);
    c->vc_cap = std::max<size_t>(2 * nvc, nvc + 4 * (c->h_sv.size() + 64));
    c->deps_cap = 2 * c->h_deps.size() + 1024;
    take(c->r_wc_off, c->h_wc_off.size() * 4);
    take(c->r_wc_cid, c->vc_cap * 4);
    take(c->r_wc_d, c->vc_cap * s);
    take(c->r_c_n, c->wc_cap * 4);
    take(c->r_c_node, c->wc_cap * kWcMaxNodes * 4);
    take(c->r_c_w, c->wc_cap * kWcMaxNodes * s);
    take(c->r_c_anchor, c->wc_cap * s4);
    take(c->r_c_K, c->wc_cap * kWcMaxNodes * s);
    take(c->r_tet_id, c->h_tet_id.size() * 16);
    take(c->r_tet_a, c->h_tet_a.size());
    take(c->r_tet_b, c->h_tet_b.size());
    take(c->r_tet_c, c->h_tet_c.size());
    take(c->r_int2orig, (size_t)std::max<int64_t>(c->n_local, 1) * 4);
    take(c->r_targets, c->h_targets.size());

    take(c->r_part_e, (size_t)c->nb * p.ge * 8);
    take(c->r_part_r, (size_t)c->nb * p.gr * 8);
    take(c->r_results, (size_t)c->nb * 2 * 8);
    take(c->r_flag, 4);
    take(c->r_mass, c->h_mass.size());

    take(c->r_halo_send, std::max<size_t>(c->h_halo_send.size(), 1) * 4);
    take(c->r_halo_recv, std::max<size_t>(c->h_halo_recv.size(), 1) * 4);
    take(c->r_dep_off, c->h_dep_off.size() * 4);
    take(c->r_deps, std::max<size_t>(c->deps_cap, 1) * 4);
    take(c->r_pipe, 8 + (size_t)c->nb * (size_t)std::max<int64_t>(c->n_chunks, 1) * 4);  // counter, flags
    take(c->r_surf, std::max<size_t>(c->h_surf.size(), 1) * 16);
    take(c->r_sv, std::max<size_t>(c->h_sv.size(), 1) * 8);
    take(c->r_chead, (size_t)std::max<int64_t>(c->prob.n_cbuckets, 1) * 4);
    take(c->r_cnext, std::max<size_t>(c->h_surf.size(), 1) * 8 * 8);  // <= 8 cells per triangle, {tri, next}
    take(c->r_cres, std::max<size_t>(c->h_sv.size(), 1) * sizeof(ContactHit));
    take(c->r_cscal, 64);
    // halo buffers of the in-library transport: Real4 [n_batch][n][3] per (colour, peer) segment
    const size_t n_send = c->halo_send_off.empty() ? 0 : (size_t)c->halo_send_off.back();
    const size_t n_recv = c->halo_recv_off.empty() ? 0 : (size_t)c->halo_recv_off.back();
    take(c->r_hsend, (size_t)c->nb * n_send * 3 * s4);
    take(c->r_hrecv, (size_t)c->nb * n_recv * 3 * s4);
    take(c->r_allred, (size_t)c->nb * 2 * 8);
    c->ws_need = off;
}

double sweep_bytes_model(const pbng_ctx *c) {
    // algorithmic HBM bytes of one iteration: pair records once (shared by the
    // samples of a batch), chunk offsets, per free vertex and sample: degree, position write, blend
    // traffic (x^{l-1} read, x^{l-1} and x^{l+1} writes) and body force; all positions read once.
    const double s = (double)c->real_size();
    // path-ordered NH records: {id | drop, VE} + {s'_0..2, det B'} = 24 B (fp32) / 48 B (fp64) per record
    // (load-only ones included) + the per-vertex first slots (8 B)
    // rest-recompute records: {id | drop, E_e/6} = 8 B (fp32) / 16 B (fp64), plus every held vertex's rest
    // position read once (below)
    // table records: {id | entry | drop, VE} (+ VE in fp64) = 8 B / 16 B, the table itself is <= 8 KB
    const double rec = (c->rest_rec || c->tab_rec) ? (c->dtype == DT_F64 ? 16.0 : 8.0)
                       : c->path_rec ? (c->dtype == DT_F64 ? 48.0 : 24.0)
                       : c->model == MODEL_NH ? (c->dtype == DT_F64 ? 56.0 : 32.0) : (c->dtype == DT_F64 ? 96.0 : 52.0);
    double b = (double)(c->path_rec ? c->n_records : c->n_pairs) * rec + (double)(c->n_chunks + 1) * 8.0 +
               (double)c->n_free * (c->path_rec ? 12.0 : 4.0);
    double per_v = 3 * s;  // write x_PBNG
    per_v += (c->prob.has_fext ? 3 * s : 0);
    b += (double)c->nb * ((double)c->n_free * per_v + (double)c->n_local * 3 * s);
    if (c->rest_rec) b += (double)c->n_local * 3 * s;
    return b;
}

double accel_bytes_model(const pbng_ctx *c) {
    return (double)c->nb * (double)c->n_free * 9.0 * (double)c->real_size();
}

// Warps per 32-vertex chunk (sweep_split_kernel / the pipelined kernel's groups), ONE value per problem so
// that both schedules and every rank of a decomposition sum each vertex's terms in the same order: the
// fixed-corotated pair (a polar decomposition) is compute-heavy, and with few chunks per colour one warp
// per chunk leaves the machine idle (the colour's dependency chain is then latency bound), so both split
// the pair loop over several warps.  PBNG_SPLIT=1|2|4 overrides (experiments).
bool batched_layout(const pbng_ctx *c) {
    static const int mode = [] {
        const char *e = getenv("PBNG_BATCHED");
        return e ? atoi(e) : 1;
    }();
    return mode != 0 && c->nb >= 32;
}

int problem_split(const pbng_ctx *c) {
    static const int forced = [] {
        const char *e = getenv("PBNG_SPLIT");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
    // rest-recompute records requested explicitly: they exist only as path records, walked by one warp per chunk
    if ((c->records == PBNG_RECORDS_REST || c->records == PBNG_RECORDS_TABLE) && c->model == MODEL_NH &&
        !batched_layout(c))
        return 1;
    int64_t gfree = 0;  // free vertices of the whole mesh (all ranks)
    for (int64_t k : c->gcol_nfree) gfree += k;
    const int64_t chunks_per_colour = gfree * c->nb / kChunk / std::max(c->ncol, 1);
    if (c->model == MODEL_FCR) return chunks_per_colour < 148 * 8 ? 8 : 4;  // config 2: 8 warps 1.17x faster
    if (chunks_per_colour < 148 * 16) return 4;
    if (chunks_per_colour < 148 * 32) return 2;
    return 1;
}

pbng_status require_device(pbng_ctx *c) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (!c->on_device()) return fail(PBNG_E_NO_DEVICE, "host-only context (device = -1)");
    return PBNG_OK;
}

cudaError_t get_event_pair(pbng_ctx *c, std::pair<cudaEvent_t, cudaEvent_t> &ev) {
    if (!c->ev_free.empty()) {
        ev = c->ev_free.back();
        c->ev_free.pop_back();
        return cudaSuccess;
    }
    cudaError_t e = cudaEventCreate(&ev.first);
    if (e != cudaSuccess) return e;
    return cudaEventCreate(&ev.second);
}

// profiling mode 1: an event pair around every sweep launch
template <class F>
cudaError_t timed_launch(pbng_ctx *c, F &&launch) {
    if (c->profiling != 1) return launch();
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    cudaError_t e = get_event_pair(c, ev);
    if (e != cudaSuccess) return e;
    cudaEventRecord(ev.first, c->stream);
    e = launch();
    cudaEventRecord(ev.second, c->stream);
    c->ev_used.push_back(ev);
    c->ev_launches.push_back(1);
    return e;
}
cudaError_t timed_sweep(pbng_ctx *c, const SweepLaunch &s) {
    return timed_launch(c, [&] { return launch_sweep(c->prob, c->L, s, c->stream); });
}

// the windowed persistent schedule of the batched fp32 NH layout (sh 6, undecomposed, <= 32 colours,
// colour launches not forced).  Auto: one window holding every sample-group pair when there are at most 8
// (n_batch <= 512 -- the per-GPU shard of config 4 at 8 GPUs), where the colour launches are short and
// their tails and launch gaps dominate (512 samples: 0.173 vs 0.202 ms per iteration); colour launches
// otherwise (4096 samples: windows of 4 / 8 / 16 take 1.72 / 1.345 / 1.33 ms against 1.147, DESIGN.md
// section 7).  PBNG_B2_WINDOW (read per call) overrides: group pairs per window, 0 = colour launches.
int b2_window_size(const pbng_ctx *c) {
    const char *e = getenv("PBNG_B2_WINDOW");
    if (e) return atoi(e);
    const int n_gp = (c->nb + 63) / 64;
    return n_gp <= 8 ? n_gp : 0;
}
bool b2_window_schedule(const pbng_ctx *c) {
    return c->prob.lane_shift == 6 && c->n_ranks == 1 && c->ncol <= kB2MaxColours && b2_window_size(c) > 0 &&
           c->schedule != PBNG_SCHEDULE_COLOUR_LAUNCHES;
}

pbng_status check_iterate(pbng_ctx *c, pbng_accel accel, double omega, double rho, double gamma, const char *who) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    const std::string w(who);
    if (!c->positions_set) return fail(PBNG_E_BAD_ORDER, w + ": set_positions first");
    if (accel != PBNG_ACCEL_NONE && accel != PBNG_ACCEL_SOR && accel != PBNG_ACCEL_CHEBYSHEV)
        return fail(PBNG_E_INVALID_ARGUMENT, w + ": unknown acceleration");
    if (accel == PBNG_ACCEL_SOR && !(omega > 0.0 && omega < 2.0))
        return fail(PBNG_E_INVALID_ARGUMENT, w + ": SOR omega must be in (0, 2)");
    if (accel == PBNG_ACCEL_CHEBYSHEV && (!(rho >= 0.0 && rho < 1.0) || !(gamma > 0.0 && gamma <= 2.0)))
        return fail(PBNG_E_INVALID_ARGUMENT, w + ": Chebyshev needs rho in [0,1) and gamma in (0,2]");
    if (accel != PBNG_ACCEL_NONE && !c->hist_valid)
        return fail(PBNG_E_BAD_ORDER, w + ": x^{l-1} was not kept by non-accelerated iterations; call set_positions");
    return PBNG_OK;
}

// one colour pass of iteration l with the blend weights of PAPER.md:605-616; part 1 =
// the colour's halo-send vertices, 2 = the others, 0 = both (one launch per non-empty part)
cudaError_t sweep_colour_impl(pbng_ctx *c, int32_t col, pbng_accel accel, double omega, double rho, double gamma,
                              int64_t *launched, int part = 0) {
    SweepLaunch s;
    s.accel = accel;
    s.work = c->work;
    s.out = c->out;
    s.hist = c->hist;
    if (accel == PBNG_ACCEL_SOR) {
        s.omega = omega;
    } else if (accel == PBNG_ACCEL_CHEBYSHEV) {
        s.omega = chebyshev_weight(c->l + 1, rho);
        s.gamma = gamma;
    }
    s.split = problem_split(c);
    // consecutive colour launches of a batched context walk the sample-group pairs in opposite orders, so
    // a launch starts on the groups whose positions the previous one left in L2
    s.reverse = col & 1;
    const int32_t ns = c->col_nsend[col];
    for (int p = 1; p <= 2; ++p) {
        if (part != 0 && part != p) continue;
        s.v_begin = c->col_vbegin[col] + (p == 1 ? 0 : ns);
        s.n_v = p == 1 ? ns : c->col_nfree[col] - ns;
        s.chunk_begin = p == 1 ? c->col_chunk[col] : c->col_chunk_mid[col];
        if (s.n_v == 0) continue;
        cudaError_t e = timed_sweep(c, s);
        if (e != cudaSuccess) return e;
        c->launches += 1;
        *launched += 1;
    }
    return cudaSuccess;
}

// after the last colour: x^{l+1} becomes the working buffer (accelerated), l += 1
void end_iteration_impl(pbng_ctx *c, pbng_accel accel) {
    if (accel != PBNG_ACCEL_NONE) std::swap(c->work, c->out);
    else c->hist_valid = false;
    c->l += 1;
    c->cur_accel = -1;
}

// Undo what apply_l2_persistence changed outside the workspace: the access-policy window on the stream it
// was set on, the persisting lines it left in L2 and the device's persisting-L2 limit.
void clear_l2_persistence(pbng_ctx *c) {
    if (!c->l2_applied) return;
    DevGuard g(c->device);
    cudaStreamAttrValue v;
    std::memset(&v, 0, sizeof(v));
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(c->l2_stream, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c->l2_prev_limit);
    c->l2_applied = false;
}

// L2 access-policy window over the gathered position buffers (pbng_set_l2_persistence)
pbng_status apply_l2_persistence(pbng_ctx *c, int enable) {
    clear_l2_persistence(c);
    if (!enable) return PBNG_OK;
    DevGuard g(c->device);
    // the two buffers the colour passes gather from (work, and out = the next iteration's work) are
    // contiguous regions of the workspace; the record stream passing through L2 is left to stream
    int max_window = 0, max_persist = 0;
    PBNG_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device), "l2: attribute");
    PBNG_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device), "l2: attribute");
    const char *base = static_cast<const char *>(c->ws) + c->r_x[0].off;
    const size_t bytes = (c->r_x[1].off + c->r_x[1].bytes) - c->r_x[0].off;
    // buffers larger than the persisting carve-out would thrash it (measured slower on config 4 and the
    // fp64 variant of config 3): no window
    if (bytes > (size_t)max_window || bytes > (size_t)max_persist) return PBNG_OK;
    size_t prev = 0;
    PBNG_CUDA(cudaDeviceGetLimit(&prev, cudaLimitPersistingL2CacheSize), "l2: persisting limit");
    PBNG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(bytes, (size_t)max_persist)),
              "l2: persisting limit");
    cudaStreamAttrValue v;
    std::memset(&v, 0, sizeof(v));
    v.accessPolicyWindow.base_ptr = const_cast<char *>(base);
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaError_t e = cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v);
    if (e != cudaSuccess) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev);
        return cuda_fail(e, "l2: stream attribute");
    }
    c->l2_applied = true;
    c->l2_stream = c->stream;
    c->l2_prev_limit = prev;
    return PBNG_OK;
}

// ------------------------------------------------------------------------------------------------
// In-library halo transport (SURVEY.md §8(b) pbng_partition, §8(e)): NCCL loaded at run time
// ------------------------------------------------------------------------------------------------

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

// libnccl.so.2 is dlopen'ed on first use: the copy PyTorch already loaded (same SONAME) is reused, so one
// process never holds two NCCLs; host-only contexts and single-GPU runs never need it.
const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char *e = dlerror();
            api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        bool all = true;
        auto sym = [&](auto &fn, const char *name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                all = false;
                api.why += std::string(" missing ") + name;
            }
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = all;
    });
    return api;
}

pbng_status nccl_fail(ncclResult_t r, const char *where) {
    const NcclApi &A = nccl();
    return fail(PBNG_E_NCCL, std::string(where) + ": " + (A.GetErrorString ? A.GetErrorString(r) : "nccl error"));
}

// byte offsets of the (colour, peer) segment in the context's halo send / receive buffers
size_t halo_seg_bytes(const pbng_ctx *c, int64_t count) { return (size_t)c->nb * (size_t)count * 3 * c->real4_size(); }
char *halo_send_buf(pbng_ctx *c, size_t seg) {
    return static_cast<char *>(c->ws) + c->r_hsend.off + halo_seg_bytes(c, c->halo_send_off[seg]);
}
char *halo_recv_buf(pbng_ctx *c, size_t seg) {
    return static_cast<char *>(c->ws) + c->r_hrecv.off + halo_seg_bytes(c, c->halo_recv_off[seg]);
}
int64_t halo_n_send(const pbng_ctx *c, size_t seg) { return c->halo_send_off[seg + 1] - c->halo_send_off[seg]; }
int64_t halo_n_recv(const pbng_ctx *c, size_t seg) { return c->halo_recv_off[seg + 1] - c->halo_recv_off[seg]; }

cudaError_t ensure_dd_streams(pbng_ctx *c) {
    if (c->dd_side) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&c->dd_side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->dd_cap, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->dd_ev_a, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->dd_ev_b, cudaEventDisableTiming);
    return e;
}

void drop_dd_graph(pbng_ctx *c) {
    if (c->dd_graph) cudaGraphExecDestroy(c->dd_graph);
    c->dd_graph = nullptr;
    c->dd_key = pbng_ctx::GraphKey();
}

// ---- peer-store halo transport: set-up (kernels: pbng_kernels.cu "Peer-store halo transport") ----

void peer_release(pbng_ctx *c) {
    pbng_ctx::PeerState &P = c->peer;
    for (auto &q : P.peer) {
        if (q.ipc_ws) cudaIpcCloseMemHandle(q.ipc_ws);
        if (q.ipc_flags) cudaIpcCloseMemHandle(q.ipc_flags);
    }
    P.peer.clear();
    P.nbr.clear();
    if (P.flags) cudaFree(P.flags);
    if (P.rows) cudaFree(P.rows);
    P.flags = nullptr;
    P.rows = nullptr;
    P.enabled = false;
}

bool peer_stale(const pbng_ctx *c) { return !c->peer.enabled || c->peer.gen != c->layout_gen || c->peer.ws != c->ws; }

// own allocations and the neighbour list (ranks with a non-empty send or receive list in some colour)
cudaError_t peer_alloc(pbng_ctx *c) {
    peer_release(c);
    pbng_ctx::PeerState &P = c->peer;
    const int n_ranks = c->n_ranks;
    P.peer.assign(n_ranks, pbng_ctx::PeerState::Peer());
    for (int q = 0; q < n_ranks; ++q) {
        if (q == c->rank) continue;
        bool any = false;
        for (int32_t col = 0; col < c->ncol && !any; ++col) {
            const size_t seg = (size_t)col * n_ranks + q;
            any = halo_n_send(c, seg) > 0 || halo_n_recv(c, seg) > 0;
        }
        if (any) P.nbr.push_back(q);
    }
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&P.flags), (size_t)(3 * n_ranks + 4) * 4);
    if (e == cudaSuccess) e = cudaMemset(P.flags, 0, (size_t)(3 * n_ranks + 4) * 4);
    const size_t n_send = c->halo_send_off.empty() ? 0 : (size_t)c->halo_send_off.back();
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&P.rows), std::max<size_t>(n_send, 1) * 4);
    return e;
}

// loopback group: the "peer mappings" are the other contexts' own device pointers
pbng_status peer_setup_group(const std::vector<pbng_ctx *> &ranks) {
    for (pbng_ctx *c : ranks) {
        PBNG_CUDA(peer_alloc(c), "peer halo: allocation");
        const int n_ranks = c->n_ranks;
        const size_t n_send = (size_t)c->halo_send_off.back();
        std::vector<int32_t> rows(std::max<size_t>(n_send, 1), 0);
        for (int q : c->peer.nbr) {
            const pbng_ctx *d = ranks[q];
            for (int32_t col = 0; col < c->ncol; ++col) {
                const size_t sseg = (size_t)col * n_ranks + q, rseg = (size_t)col * n_ranks + c->rank;
                const int64_t n = halo_n_send(c, sseg);
                if (n != halo_n_recv(d, rseg))
                    return fail(PBNG_E_INVALID_ARGUMENT, "peer halo: send and receive lists of two ranks differ in length");
                for (int64_t k = 0; k < n; ++k) {
                    // the k-th vertex rank c sends is the k-th vertex rank q receives (both ascending original id)
                    if (c->halo_send_orig[c->halo_send_off[sseg] + k] != d->halo_recv_orig[d->halo_recv_off[rseg] + k])
                        return fail(PBNG_E_INVALID_ARGUMENT, "peer halo: send and receive lists of two ranks differ");
                    rows[c->halo_send_off[sseg] + k] = d->h_halo_recv[d->halo_recv_off[rseg] + k];
                }
            }
        }
        PBNG_CUDA(cudaMemcpy(c->peer.rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice), "peer halo: rows");
    }
    for (pbng_ctx *c : ranks) {
        for (int q : c->peer.nbr) {
            pbng_ctx *d = ranks[q];
            pbng_ctx::PeerState::Peer &P = c->peer.peer[q];
            for (int k = 0; k < 3; ++k) P.x[k] = d->L.xbuf[k];
            P.stride = d->prob.x_stride;
            P.sh = d->prob.lane_shift;
            P.n_local = d->n_local;
            P.flags = d->peer.flags;
        }
        c->peer.enabled = true;
        c->peer.gen = c->layout_gen;
        c->peer.ws = c->ws;
    }
    return PBNG_OK;
}

// what a rank tells the others about its memory (all-gathered through the communicator)
struct PeerHello {
    cudaIpcMemHandle_t ws, flags;
    uint64_t ws_off;     // the workspace's offset inside the allocation the handle names
    uint64_t x_off[3];   // position buffers, bytes from the workspace base
    int64_t x_stride;
    int32_t sh, pad;
    int64_t n_local;     // vertices this rank holds
};

// one process per GPU: IPC handles of the workspace allocation and the flag words, and the neighbours'
// ghost rows, exchanged over the context's NCCL communicator (collective)
pbng_status peer_setup_comm(pbng_ctx *c) {
    const NcclApi &A = nccl();
    PBNG_CUDA(peer_alloc(c), "peer halo: allocation");
    const int n_ranks = c->n_ranks;
    PeerHello me;
    std::memset(&me, 0, sizeof(me));
    // the bound workspace is usually a slice of a caching allocator's block: the handle names the whole
    // cudaMalloc allocation, the slice is found by its offset (cuMemGetAddressRange through the runtime)
    typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    PBNG_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &qr), "peer halo: driver entry point");
    if (!fn || qr != cudaDriverEntryPointSuccess) return fail(PBNG_E_CUDA, "peer halo: cuMemGetAddressRange not available");
    unsigned long long base = 0;
    size_t size = 0;
    if (reinterpret_cast<GetRange>(fn)(&base, &size, (unsigned long long)(uintptr_t)c->ws) != 0)
        return fail(PBNG_E_CUDA, "peer halo: the workspace is not a device allocation");
    PBNG_CUDA(cudaIpcGetMemHandle(&me.ws, reinterpret_cast<void *>((uintptr_t)base)),
              "peer halo: cudaIpcGetMemHandle(workspace) -- allocate the workspace with cudaMalloc (PyTorch: not "
              "expandable_segments)");
    PBNG_CUDA(cudaIpcGetMemHandle(&me.flags, c->peer.flags), "peer halo: cudaIpcGetMemHandle(flags)");
    me.ws_off = (uint64_t)((uintptr_t)c->ws - (uintptr_t)base);
    for (int k = 0; k < 3; ++k) me.x_off[k] = (uint64_t)(static_cast<char *>(c->L.xbuf[k]) - static_cast<char *>(c->ws));
    me.x_stride = c->prob.x_stride;
    me.sh = c->prob.lane_shift;
    me.n_local = c->n_local;
    PeerHello *d_all = nullptr;
    PBNG_CUDA(cudaMalloc(reinterpret_cast<void **>(&d_all), sizeof(PeerHello) * (size_t)n_ranks), "peer halo: allocation");
    std::vector<PeerHello> all(n_ranks);
    pbng_status st = PBNG_OK;
    do {
        cudaError_t e = cudaMemcpyAsync(d_all + c->rank, &me, sizeof(me), cudaMemcpyHostToDevice, c->stream);
        if (e != cudaSuccess) { st = cuda_fail(e, "peer halo: copy"); break; }
        ncclResult_t r = A.AllGather(d_all + c->rank, d_all, sizeof(PeerHello), ncclUint8, c->comm, c->stream);
        if (r != ncclSuccess) { st = nccl_fail(r, "peer halo: all-gather"); break; }
        // the neighbours' ghost rows: rank q's receive list (colour, this rank) is this rank's row list (colour, q)
        r = A.GroupStart();
        for (int q : c->peer.nbr)
            for (int32_t col = 0; col < c->ncol && r == ncclSuccess; ++col) {
                const size_t seg = (size_t)col * n_ranks + q;
                const int64_t ns = halo_n_send(c, seg), nr = halo_n_recv(c, seg);
                if (nr > 0) r = A.Send(c->L.halo_recv + c->halo_recv_off[seg], (size_t)nr * 4, ncclUint8, q, c->comm, c->stream);
                if (r == ncclSuccess && ns > 0)
                    r = A.Recv(c->peer.rows + c->halo_send_off[seg], (size_t)ns * 4, ncclUint8, q, c->comm, c->stream);
            }
        ncclResult_t r2 = A.GroupEnd();
        if (r == ncclSuccess) r = r2;
        if (r != ncclSuccess) { st = nccl_fail(r, "peer halo: row exchange"); break; }
        e = cudaMemcpyAsync(all.data(), d_all, sizeof(PeerHello) * (size_t)n_ranks, cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) { st = cuda_fail(e, "peer halo: exchange"); break; }
    } while (false);
    cudaFree(d_all);
    if (st != PBNG_OK) return st;
    for (int q : c->peer.nbr) {
        pbng_ctx::PeerState::Peer &P = c->peer.peer[q];
        PBNG_CUDA(cudaIpcOpenMemHandle(&P.ipc_ws, all[q].ws, cudaIpcMemLazyEnablePeerAccess),
                  "peer halo: cudaIpcOpenMemHandle(workspace) -- the ranks' GPUs need peer access (NVLink / NVSwitch)");
        PBNG_CUDA(cudaIpcOpenMemHandle(&P.ipc_flags, all[q].flags, cudaIpcMemLazyEnablePeerAccess),
                  "peer halo: cudaIpcOpenMemHandle(flags)");
        char *ws = static_cast<char *>(P.ipc_ws) + all[q].ws_off;
        for (int k = 0; k < 3; ++k) P.x[k] = ws + all[q].x_off[k];
        P.stride = all[q].x_stride;
        P.sh = all[q].sh;
        P.n_local = all[q].n_local;
        P.flags = static_cast<uint32_t *>(P.ipc_flags);
    }
    c->peer.enabled = true;
    c->peer.gen = c->layout_gen;
    c->peer.ws = c->ws;
    return PBNG_OK;
}

// The exchange step of one colour, on stream `side`, after every rank's part-1 vertices of the colour
// are final: pack each (rank, peer) send list, move the buffers, unpack each receive list.  `ranks` are
// the rank contexts this process drives (one with NCCL, all of them in the loopback group).
struct Exchange {
    std::vector<pbng_ctx *> ranks;
    bool loopback = false;
    bool peer = false;  // peer-store transport: rows stored straight into the neighbours' ghost rows

    static uint64_t peer_timeout_ns() {
        const char *e = getenv("PBNG_PEER_TIMEOUT_MS");
        const long ms = e ? atol(e) : 20000;
        return (uint64_t)(ms > 0 ? ms : 20000) * 1000000ull;
    }
    // flag words of a rank: pushed[q] at q, done[q] at n_ranks + q, block counter of the push to q at 2 n_ranks + q
    // start of an iterate block: zero the flag words; between processes a barrier keeps a fast neighbour's
    // first signal from landing before the zeroing
    cudaError_t peer_begin(cudaStream_t main) {
        for (pbng_ctx *c : ranks) {
            cudaError_t e = cudaMemsetAsync(c->peer.flags, 0, (size_t)(3 * c->n_ranks + 4) * 4, main);
            if (e != cudaSuccess) return e;
        }
        if (!loopback) {
            pbng_ctx *c = ranks[0];
            uint32_t *scratch = c->peer.flags + 3 * c->n_ranks;
            ncclResult_t r = nccl().AllReduce(scratch, scratch, 1, ncclInt32, ncclSum, c->comm, main);
            if (r != ncclSuccess) {
                status = nccl_fail(r, "iterate: peer-halo barrier");
                return cudaErrorUnknown;
            }
        }
        return cudaSuccess;
    }
    // end of pass E (colour col; both parts and the pushes are in stream order before this), ONE launch per
    // rank: tell every neighbour this rank is done reading pass E, then wait for the rows the neighbours
    // stored during pass E -- pass E + 1 reads them
    cudaError_t peer_sync(int32_t col, uint32_t E, cudaStream_t main) {
        for (pbng_ctx *c : ranks) {
            PeerSignal S;
            S.val = E;
            for (int q : c->peer.nbr) S.flag[S.n++] = c->peer.peer[q].flags + c->n_ranks + c->rank;
            PeerWait W;
            W.flags = c->peer.flags;
            W.want = E;
            W.timeout_ns = peer_timeout_ns();
            for (int q : c->peer.nbr)
                if (halo_n_recv(c, (size_t)col * c->n_ranks + q) > 0) W.slot[W.n++] = q;
            if (S.n == 0 && W.n == 0) continue;
            cudaError_t e = launch_halo_sync(c->L, S, W, main);
            if (e != cudaSuccess) return e;
            ++launches;
        }
        return cudaSuccess;
    }
    // the exchange of pass E (colour col) on `side`: per neighbour ONE kernel { wait done >= E - 1; store rows;
    // pushed = E }
    cudaError_t run_peer(int32_t col, int nf, uint32_t E, cudaStream_t side) {
        for (pbng_ctx *c : ranks) {
            const int n_ranks = c->n_ranks;
            for (int q : c->peer.nbr) {
                const size_t seg = (size_t)col * n_ranks + q;
                const int64_t n = halo_n_send(c, seg);
                if (n == 0) continue;
                const pbng_ctx::PeerState::Peer &P = c->peer.peer[q];
                PeerPush A;
                A.idx = c->L.halo_send + c->halo_send_off[seg];
                A.rows = c->peer.rows + c->halo_send_off[seg];
                A.n = n;
                A.nf = nf;
                A.buf[0] = c->work;
                A.buf[1] = c->out;
                A.buf[2] = c->hist;
                A.x_stride = c->prob.x_stride;
                A.sh = c->prob.lane_shift;
                for (int k = 0; k < 3; ++k) A.peer_x[k] = P.x[k];
                A.peer_stride = P.stride;
                A.peer_sh = P.sh;
                A.peer_n_vertices = P.n_local;
                A.wait_flag = c->peer.flags + n_ranks + q;
                A.wait_val = E - 1;
                A.sig_flag = P.flags + c->rank;
                A.sig_val = E;
                A.counter = c->peer.flags + 2 * n_ranks + q;
                A.timeout_ns = peer_timeout_ns();
                cudaError_t e = launch_halo_push(c->prob, c->L, A, side);
                if (e != cudaSuccess) return e;
                ++launches;
            }
        }
        return cudaSuccess;
    }
    // after pass E (both parts and the pushes): tell every neighbour this rank is done reading pass E
    cudaError_t peer_signal_done(uint32_t E, cudaStream_t main) {
        for (pbng_ctx *c : ranks) {
            PeerSignal S;
            S.val = E;
            for (int q : c->peer.nbr) S.flag[S.n++] = c->peer.peer[q].flags + c->n_ranks + c->rank;
            if (S.n == 0) continue;
            cudaError_t e = launch_halo_signal(S, main);
            if (e != cudaSuccess) return e;
            ++launches;
        }
        return cudaSuccess;
    }
    // end of the block: every neighbour is through its last pass (its rows of that pass landed before its
    // done signal), so nothing more is stored here
    cudaError_t peer_end(uint32_t E_last, cudaStream_t main) {
        if (E_last == 0) return cudaSuccess;
        for (pbng_ctx *c : ranks) {
            PeerWait W;
            W.flags = c->peer.flags;
            W.want = E_last;
            W.timeout_ns = peer_timeout_ns();
            for (int q : c->peer.nbr) W.slot[W.n++] = c->n_ranks + q;
            if (W.n == 0) continue;
            cudaError_t e = launch_halo_wait(c->L, W, main);
            if (e != cudaSuccess) return e;
            ++launches;
        }
        return cudaSuccess;
    }
    int64_t launches = 0;
    pbng_status status = PBNG_OK;

    cudaError_t run(int32_t col, int nf, cudaStream_t side) {
        const int n_ranks = ranks[0]->n_ranks;
        for (pbng_ctx *c : ranks) {
            const int bufs[3] = {c->work, c->out, c->hist};
            for (int p = 0; p < n_ranks; ++p) {
                const size_t seg = (size_t)col * n_ranks + p;
                const int64_t n = p == c->rank ? 0 : halo_n_send(c, seg);
                if (n == 0) continue;
                cudaError_t e = launch_halo_pack(c->prob, c->L, c->L.halo_send + c->halo_send_off[seg], n, nf, bufs,
                                                 halo_send_buf(c, seg), side);
                if (e != cudaSuccess) return e;
                ++launches;
            }
        }
        if (loopback) {
            for (pbng_ctx *q : ranks)  // q sends to p: p's receive segment (col, q) <- q's send segment (col, p)
                for (pbng_ctx *p : ranks) {
                    if (p == q) continue;
                    const size_t sseg = (size_t)col * n_ranks + p->rank, rseg = (size_t)col * n_ranks + q->rank;
                    const int64_t n = halo_n_send(q, sseg);
                    if (n == 0) continue;
                    cudaError_t e = cudaMemcpyAsync(halo_recv_buf(p, rseg), halo_send_buf(q, sseg),
                                                    (size_t)q->nb * n * nf * q->real4_size(), cudaMemcpyDeviceToDevice,
                                                    side);
                    if (e != cudaSuccess) return e;
                }
        } else {
            pbng_ctx *c = ranks[0];
            const NcclApi &A = nccl();
            bool any = false;
            for (int p = 0; p < n_ranks && !any; ++p)
                if (p != c->rank) {
                    const size_t seg = (size_t)col * n_ranks + p;
                    any = halo_n_send(c, seg) > 0 || halo_n_recv(c, seg) > 0;
                }
            if (any) {
                ncclResult_t r = A.GroupStart();
                for (int p = 0; p < n_ranks && r == ncclSuccess; ++p) {
                    if (p == c->rank) continue;
                    const size_t seg = (size_t)col * n_ranks + p;
                    const int64_t ns = halo_n_send(c, seg), nr = halo_n_recv(c, seg);
                    if (ns > 0)
                        r = A.Send(halo_send_buf(c, seg), (size_t)c->nb * ns * nf * c->real4_size(), ncclUint8, p,
                                   c->comm, side);
                    if (r == ncclSuccess && nr > 0)
                        r = A.Recv(halo_recv_buf(c, seg), (size_t)c->nb * nr * nf * c->real4_size(), ncclUint8, p,
                                   c->comm, side);
                }
                ncclResult_t r2 = A.GroupEnd();
                if (r == ncclSuccess) r = r2;
                if (r != ncclSuccess) {
                    status = nccl_fail(r, "iterate: halo exchange");
                    return cudaErrorUnknown;
                }
            }
        }
        for (pbng_ctx *c : ranks) {
            const int bufs[3] = {c->work, c->out, c->hist};
            for (int p = 0; p < n_ranks; ++p) {
                const size_t seg = (size_t)col * n_ranks + p;
                const int64_t n = p == c->rank ? 0 : halo_n_recv(c, seg);
                if (n == 0) continue;
                cudaError_t e = launch_halo_unpack(c->prob, c->L, c->L.halo_recv + c->halo_recv_off[seg], n, nf, bufs,
                                                   halo_recv_buf(c, seg), side);
                if (e != cudaSuccess) return e;
                ++launches;
            }
        }
        return cudaSuccess;
    }
};

// n decomposed PBNG iterations of the rank contexts `X.ranks` (PAPER.md:693-705 colour order), every
// launch on `main` except the exchange on `side`: per colour, part 1 (halo-send vertices) of every rank
// -> fork -> [side: pack, exchange, unpack] || [main: part 2 of every rank] -> join.  Packing reads only
// part-1 rows and unpacking writes only ghost rows of the colour, which no vertex of the colour reads,
// so the result is that of the serial order bit for bit (tests/test_gpu_dd.py).
cudaError_t dd_iterations(Exchange &X, cudaStream_t main, cudaStream_t side, cudaEvent_t ev_a, cudaEvent_t ev_b,
                          int32_t n, pbng_accel accel, double omega, double rho, double gamma, int64_t *sweeps) {
    const int nf = accel == PBNG_ACCEL_NONE ? 1 : 3;
    const int32_t ncol = X.ranks[0]->ncol;
    if (X.peer) {
        cudaError_t e = X.peer_begin(main);
        if (e != cudaSuccess) return e;
    }
    uint32_t E = 0;  // pass epoch of the peer-store flags: 1 + pass index within this block
    for (int32_t it = 0; it < n; ++it) {
        for (int32_t col = 0; col < ncol; ++col) {
            ++E;
            for (pbng_ctx *c : X.ranks) {
                cudaError_t e = sweep_colour_impl(c, col, accel, omega, rho, gamma, sweeps, 1);
                if (e != cudaSuccess) return e;
            }
            cudaError_t e = cudaEventRecord(ev_a, main);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_a, 0);
            if (e == cudaSuccess) e = X.peer ? X.run_peer(col, nf, E, side) : X.run(col, nf, side);
            if (e == cudaSuccess) e = cudaEventRecord(ev_b, side);
            if (e != cudaSuccess) return e;
            for (pbng_ctx *c : X.ranks) {
                e = sweep_colour_impl(c, col, accel, omega, rho, gamma, sweeps, 2);
                if (e != cudaSuccess) return e;
            }
            e = cudaStreamWaitEvent(main, ev_b, 0);
            // the block's last pass signals first and waits in a second round (peer_end): in the one-GPU
            // loopback group a rank's wait must not precede, in stream order, the signal it waits for
            if (e == cudaSuccess && X.peer)
                e = (it == n - 1 && col == ncol - 1) ? X.peer_signal_done(E, main) : X.peer_sync(col, E, main);
            if (e != cudaSuccess) return e;
        }
        for (pbng_ctx *c : X.ranks) end_iteration_impl(c, accel);
    }
    if (X.peer) return X.peer_end(E, main);
    return cudaSuccess;
}

// PBNG_DD_GRAPH=0 runs the decomposed iterations as direct launches (read per call: tests compare both)
bool dd_graphs_enabled() {
    const char *e = getenv("PBNG_DD_GRAPH");
    return !(e && atoi(e) == 0);
}

// Run dd_iterations through a CUDA graph cached on `owner` (captured on the first call from a given state,
// replayed afterwards); state = the host-side iteration state the captured launches bake in.  Falls back
// to direct launches if the capture is refused.
pbng_status dd_run(pbng_ctx *owner, Exchange &X, cudaStream_t main, cudaStream_t side, cudaStream_t cap,
                   cudaEvent_t ev_a, cudaEvent_t ev_b, int32_t n, pbng_accel accel, double omega, double rho,
                   double gamma, int64_t *sweeps, const char *who) {
    pbng_ctx::GraphKey key;
    key.n = n;
    key.accel = (int)accel;
    key.omega = accel == PBNG_ACCEL_SOR ? omega : 0.0;
    key.rho = accel == PBNG_ACCEL_CHEBYSHEV ? rho : 0.0;
    key.gamma = accel == PBNG_ACCEL_CHEBYSHEV ? gamma : 0.0;
    key.l = owner->l;
    key.work = owner->work;
    key.out = owner->out;
    key.hist = owner->hist;
    key.hist_valid = owner->hist_valid;
    key.ws = owner->ws;
    key.stream = main;
    key.inv_dt2 = owner->prob.inv_dt2;
    for (pbng_ctx *c : X.ranks) {
        key.gens.push_back(c->layout_gen);
        key.gens.push_back(reinterpret_cast<uintptr_t>(c->ws));
        key.gens.push_back((uint64_t)c->work | (uint64_t)c->l << 8);
    }
    key.gens.push_back(X.peer ? 1 : 0);
    const bool use_graph = dd_graphs_enabled() && owner->profiling != 1 && n > 0;
    if (use_graph && owner->dd_graph && owner->dd_key == key) {
        PBNG_CUDA(cudaGraphLaunch(owner->dd_graph, main), who);
        for (int32_t it = 0; it < n; ++it)
            for (pbng_ctx *c : X.ranks) end_iteration_impl(c, accel);
        for (pbng_ctx *c : X.ranks) c->launches += owner->dd_graph_launches / (int64_t)X.ranks.size();
        *sweeps += owner->dd_graph_sweeps;
        owner->dd_graph_replays += 1;
        return PBNG_OK;
    }
    if (use_graph) {
        drop_dd_graph(owner);
        // capture from a copy of the host state; the live state advances only when the graph is launched
        struct Saved {
            int work, out, hist;
            int64_t l, launches;
            bool hist_valid;
            int cur_accel;
        };
        std::vector<Saved> saved;
        for (pbng_ctx *c : X.ranks) saved.push_back({c->work, c->out, c->hist, c->l, c->launches, c->hist_valid, c->cur_accel});
        const int64_t x0 = X.launches;
        int64_t sw = 0;
        // capture on the library's own stream `cap` (the caller's may be the legacy default stream, which
        // cannot be captured), with the caller stream's L2 access-policy window copied onto it, then launch
        // the graph in the caller's stream order
        cudaStreamAttrValue win;
        std::memset(&win, 0, sizeof(win));
        if (cudaStreamGetAttribute(main, cudaStreamAttributeAccessPolicyWindow, &win) == cudaSuccess)
            cudaStreamSetAttribute(cap, cudaStreamAttributeAccessPolicyWindow, &win);
        cudaGetLastError();
        std::vector<cudaStream_t> own_streams;
        for (pbng_ctx *c : X.ranks) {
            own_streams.push_back(c->stream);
            c->stream = cap;
        }
        cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
        if (e == cudaSuccess) {
            cudaError_t ei = dd_iterations(X, cap, side, ev_a, ev_b, n, accel, omega, rho, gamma, &sw);
            cudaGraph_t graph = nullptr;
            cudaError_t ee = cudaStreamEndCapture(cap, &graph);
            for (size_t k = 0; k < X.ranks.size(); ++k) X.ranks[k]->stream = own_streams[k];
            cudaGraphExec_t exec = nullptr;
            if (ei == cudaSuccess && ee == cudaSuccess && graph)
                e = cudaGraphInstantiate(&exec, graph, 0);
            else
                e = ei != cudaSuccess ? ei : (ee != cudaSuccess ? ee : cudaErrorStreamCaptureInvalidated);
            if (graph) cudaGraphDestroy(graph);
            int64_t launched = X.launches - x0;
            for (size_t k = 0; k < X.ranks.size(); ++k) {
                pbng_ctx *c = X.ranks[k];
                launched += c->launches - saved[k].launches;
                c->work = saved[k].work;
                c->out = saved[k].out;
                c->hist = saved[k].hist;
                c->l = saved[k].l;
                c->launches = saved[k].launches;
                c->hist_valid = saved[k].hist_valid;
                c->cur_accel = saved[k].cur_accel;
            }
            if (X.status != PBNG_OK) return X.status;
            if (e == cudaSuccess) {
                owner->dd_graph = exec;
                owner->dd_key = key;
                owner->dd_graph_launches = launched;
                owner->dd_graph_sweeps = sw;
                PBNG_CUDA(cudaGraphLaunch(exec, main), who);
                for (int32_t it = 0; it < n; ++it)
                    for (pbng_ctx *c : X.ranks) end_iteration_impl(c, accel);
                for (pbng_ctx *c : X.ranks) c->launches += launched / (int64_t)X.ranks.size();
                *sweeps += sw;
                return PBNG_OK;
            }
            cudaGetLastError();  // capture refused: run the same launches directly
        } else {
            for (size_t k = 0; k < X.ranks.size(); ++k) X.ranks[k]->stream = own_streams[k];
            cudaGetLastError();
        }
    }
    cudaError_t e = dd_iterations(X, main, side, ev_a, ev_b, n, accel, omega, rho, gamma, sweeps);
    if (X.status != PBNG_OK) return X.status;
    PBNG_CUDA(e, who);
    for (pbng_ctx *c : X.ranks) c->launches += X.launches / (int64_t)X.ranks.size();
    return PBNG_OK;
}

}  // namespace

extern "C" {

const char *pbng_last_error(void) { return g_err.c_str(); }

int32_t pbng_version(void) { return 100; }

pbng_status pbng_create_mesh(const double *rest_xyz, int64_t n_vertices, const int32_t *tets, int64_t n_tets,
                             int32_t n_batch, pbng_dtype dtype, int device, uintptr_t cuda_stream, pbng_ctx **out,
                             int64_t *bad_index) {
    if (bad_index) *bad_index = -1;
    if (!out) return fail(PBNG_E_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    if (!rest_xyz || n_vertices <= 0 || n_vertices > INT32_MAX - 64 || n_tets < 0 || (n_tets > 0 && !tets) ||
        n_batch < 1 || (dtype != PBNG_F32 && dtype != PBNG_F64) || device < -1)
        return fail(PBNG_E_INVALID_ARGUMENT, "create_mesh: bad sizes, pointers, dtype or device");
    if (device >= 0) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n)
            return fail(PBNG_E_CUDA, "create_mesh: CUDA device " + std::to_string(device) + " not available");
    }
    for (int64_t k = 0; k < n_vertices * 3; ++k)
        if (!std::isfinite(rest_xyz[k])) return fail(PBNG_E_INVALID_ARGUMENT, "create_mesh: non-finite rest position");
    for (int64_t e = 0; e < n_tets; ++e)
        for (int a = 0; a < 4; ++a)
            if (tets[4 * e + a] < 0 || tets[4 * e + a] >= n_vertices) {
                if (bad_index) *bad_index = e;
                return fail(PBNG_E_INDEX_OUT_OF_RANGE, "create_mesh: tet " + std::to_string(e) + " has a vertex out of range");
            }
    pbng_ctx *c = new (std::nothrow) pbng_ctx();
    if (!c) return fail(PBNG_E_OUT_OF_MEMORY, "create_mesh: host allocation");
    try {
        c->nv = n_vertices;
        c->nt = n_tets;
        c->nb = n_batch;
        c->dtype = dtype;
        c->device = device;
        c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
        c->prob.device = device >= 0 ? device : 0;
        if (device >= 0) cudaDeviceGetAttribute(&c->prob.sm_count, cudaDevAttrMultiProcessorCount, device);
        c->X.assign(rest_xyz, rest_xyz + 3 * n_vertices);
        c->tets.assign(tets, tets + 4 * n_tets);
        c->Bm.resize((size_t)n_tets * 9);
        c->V.resize((size_t)n_tets);
        // rest precompute: Dm = [X1-X0, X2-X0, X3-X0], B = Dm^{-1}, V = |det Dm| / 6
        for (int64_t e = 0; e < n_tets; ++e) {
            const int32_t *t = tets + 4 * e;
            double Dm[9], ell = 0.0;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) Dm[3 * a + b] = c->X[3 * t[b + 1] + a] - c->X[3 * t[0] + a];
            static const int pa[6] = {0, 0, 0, 1, 1, 2}, pb[6] = {1, 2, 3, 2, 3, 3};
            for (int q = 0; q < 6; ++q) {
                double d2 = 0;
                for (int b = 0; b < 3; ++b) {
                    const double d = c->X[3 * t[pa[q]] + b] - c->X[3 * t[pb[q]] + b];
                    d2 += d * d;
                }
                ell += std::sqrt(d2) / 6.0;
            }
            const double det = det3(Dm);
            if (!(std::fabs(det) > 1e-12 * ell * ell * ell)) {
                delete c;
                if (bad_index) *bad_index = e;
                return fail(PBNG_E_DEGENERATE_ELEMENT, "create_mesh: tet " + std::to_string(e) + " is degenerate");
            }
            const double inv = 1.0 / det;
            double *B = c->Bm.data() + 9 * e;
            // inverse = adjugate / det (adjugate = transpose of the cofactor matrix)
            B[0] = (Dm[4] * Dm[8] - Dm[5] * Dm[7]) * inv;
            B[1] = (Dm[2] * Dm[7] - Dm[1] * Dm[8]) * inv;
            B[2] = (Dm[1] * Dm[5] - Dm[2] * Dm[4]) * inv;
            B[3] = (Dm[5] * Dm[6] - Dm[3] * Dm[8]) * inv;
            B[4] = (Dm[0] * Dm[8] - Dm[2] * Dm[6]) * inv;
            B[5] = (Dm[2] * Dm[3] - Dm[0] * Dm[5]) * inv;
            B[6] = (Dm[3] * Dm[7] - Dm[4] * Dm[6]) * inv;
            B[7] = (Dm[1] * Dm[6] - Dm[0] * Dm[7]) * inv;
            B[8] = (Dm[0] * Dm[4] - Dm[1] * Dm[3]) * inv;
            c->V[e] = std::fabs(det) / 6.0;
        }
    } catch (const std::bad_alloc &) {
        delete c;
        return fail(PBNG_E_OUT_OF_MEMORY, "create_mesh: host allocation");
    }
    *out = c;
    return PBNG_OK;
}

pbng_status pbng_set_material(pbng_ctx *c, pbng_model model, const double *E, int64_t n_E, double nu, double density,
                              const double gravity[3]) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (model != PBNG_NEOHOOKEAN && model != PBNG_FIXED_COROTATED && model != PBNG_STABLE_NEOHOOKEAN)
        return fail(PBNG_E_INVALID_ARGUMENT, "set_material: unknown model");
    if (!E || (n_E != 1 && n_E != c->nt)) return fail(PBNG_E_INVALID_ARGUMENT, "set_material: E must have 1 or n_tets entries");
    for (int64_t k = 0; k < n_E; ++k)
        if (!(E[k] > 0.0) || !std::isfinite(E[k])) return fail(PBNG_E_INVALID_ARGUMENT, "set_material: E must be positive and finite");
    if (!(nu >= 0.0 && nu < 0.5)) return fail(PBNG_E_INVALID_ARGUMENT, "set_material: nu must be in [0, 0.5)");
    if (!(density >= 0.0) || !std::isfinite(density)) return fail(PBNG_E_INVALID_ARGUMENT, "set_material: density must be >= 0");
    double g[3] = {0, 0, 0};
    if (gravity)
        for (int k = 0; k < 3; ++k) {
            if (!std::isfinite(gravity[k])) return fail(PBNG_E_INVALID_ARGUMENT, "set_material: non-finite gravity");
            g[k] = gravity[k];
        }
    try {
        c->E.assign(E, E + n_E);
    } catch (const std::bad_alloc &) {
        return fail(PBNG_E_OUT_OF_MEMORY, "set_material: host allocation");
    }
    c->model = model;
    c->nu = nu;
    c->density = density;
    for (int k = 0; k < 3; ++k) c->grav[k] = g[k];
    c->has_material = true;
    c->invalidate_colouring();
    return PBNG_OK;
}

pbng_status pbng_set_constraints(pbng_ctx *c, const int32_t *pinned, int64_t n_pinned, const double *pinned_xyz,
                                 const pbng_weak_constraint *wc, int64_t n_wc) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (n_pinned < 0 || n_pinned > c->nv || (n_pinned > 0 && (!pinned || !pinned_xyz)) || n_wc < 0 || (n_wc > 0 && !wc))
        return fail(PBNG_E_INVALID_ARGUMENT, "set_constraints: bad sizes or pointers");
    std::vector<char> seen((size_t)c->nv, 0);
    for (int64_t k = 0; k < n_pinned; ++k) {
        if (pinned[k] < 0 || pinned[k] >= c->nv) return fail(PBNG_E_INDEX_OUT_OF_RANGE, "set_constraints: pinned vertex out of range");
        if (seen[pinned[k]]) return fail(PBNG_E_INVALID_ARGUMENT, "set_constraints: duplicate pinned vertex");
        seen[pinned[k]] = 1;
    }
    for (int64_t k = 0; k < (int64_t)c->nb * n_pinned * 3; ++k)
        if (!std::isfinite(pinned_xyz[k])) return fail(PBNG_E_INVALID_ARGUMENT, "set_constraints: non-finite target");
    {
        pbng_status st = validate_wc(c, wc, n_wc, "set_constraints");
        if (st != PBNG_OK) return st;
    }
    try {
        std::vector<int64_t> order((size_t)n_pinned);
        for (int64_t k = 0; k < n_pinned; ++k) order[k] = k;
        std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return pinned[a] < pinned[b]; });
        c->pin_order = order;
        c->pinned.resize((size_t)n_pinned);
        c->targets.resize((size_t)c->nb * n_pinned * 3);
        for (int64_t k = 0; k < n_pinned; ++k) {
            c->pinned[k] = pinned[order[k]];
            for (int64_t b = 0; b < c->nb; ++b)
                for (int a = 0; a < 3; ++a)
                    c->targets[3 * (b * n_pinned + k) + a] = pinned_xyz[3 * (b * n_pinned + order[k]) + a];
        }
        c->wc.assign(wc, wc + n_wc);
    } catch (const std::bad_alloc &) {
        return fail(PBNG_E_OUT_OF_MEMORY, "set_constraints: host allocation");
    }
    c->has_constraints = true;
    c->invalidate_colouring();
    return PBNG_OK;
}

// colouring (greedy, or `given` -- the incremental recolouring of pbng_update_constraints) and the
// colour-sorted device layout it implies
// vertex -> incident tets in ascending tet index (CSR), cached in the context (the mesh never changes)
static void incidence(pbng_ctx *c) {
    const int64_t nv = c->nv, nt = c->nt;
    c->inc_off.assign((size_t)nv + 1, 0);
    for (int64_t e = 0; e < nt; ++e)
        for (int a = 0; a < 4; ++a) c->inc_off[c->tets[4 * e + a] + 1]++;
    for (int64_t v = 0; v < nv; ++v) c->inc_off[v + 1] += c->inc_off[v];
    c->inc.assign((size_t)std::max<int64_t>(c->inc_off[nv], 1), 0);
    std::vector<int64_t> fill(c->inc_off.begin(), c->inc_off.end() - 1);
    for (int64_t e = 0; e < nt; ++e)
        for (int a = 0; a < 4; ++a) c->inc[fill[c->tets[4 * e + a]]++] = (int32_t)e;
}

static pbng_status colour_and_layout(pbng_ctx *c, const std::vector<int32_t> *given) {
    drop_dd_graph(c);
    c->layout_gen += 1;
    PhaseTimer T;
    try {
        const int64_t nv = c->nv, nt = c->nt, nwc = (int64_t)c->wc.size();
        // vertex -> incident tets (ascending tet index) and vertex -> stencils (tets, then constraints)
        if (c->inc_off.empty()) incidence(c);
        const std::vector<int64_t> &vt_off = c->inc_off;
        const std::vector<int32_t> &vt = c->inc;
        std::vector<int64_t> vs_off((size_t)nv + 1, 0);
        std::vector<std::vector<int32_t>> cnodes((size_t)nwc);
        for (int64_t q = 0; q < nwc; ++q) {
            const pbng_weak_constraint &w = c->wc[q];
            for (int a = 0; a < w.n0; ++a) cnodes[q].push_back(w.idx0[a]);
            for (int a = 0; a < w.n1; ++a) cnodes[q].push_back(w.idx1[a]);
            std::sort(cnodes[q].begin(), cnodes[q].end());
            cnodes[q].erase(std::unique(cnodes[q].begin(), cnodes[q].end()), cnodes[q].end());
        }
        std::vector<int64_t> vc_cnt((size_t)nv, 0);
        for (int64_t q = 0; q < nwc; ++q)
            for (int32_t v : cnodes[q]) vc_cnt[v]++;
        for (int64_t v = 0; v < nv; ++v) vs_off[v + 1] = vs_off[v] + (vt_off[v + 1] - vt_off[v]) + vc_cnt[v];
        std::vector<int64_t> vs((size_t)std::max<int64_t>(vs_off[nv], 1));
        {
            std::vector<int64_t> fill(vs_off.begin(), vs_off.end() - 1);
            for (int64_t v = 0; v < nv; ++v)
                for (int64_t k = vt_off[v]; k < vt_off[v + 1]; ++k) vs[fill[v]++] = vt[k];
            for (int64_t q = 0; q < nwc; ++q)
                for (int32_t v : cnodes[q]) vs[fill[v]++] = nt + q;
        }
        // isolated free vertices make A singular
        std::vector<char> is_pinned((size_t)nv, 0);
        for (int32_t p : c->pinned) is_pinned[p] = 1;
        for (int64_t v = 0; v < nv; ++v)
            if (!is_pinned[v] && vs_off[v + 1] == vs_off[v])
                return fail(PBNG_E_ISOLATED_VERTEX, "color: free vertex " + std::to_string(v) + " has no element or constraint");
        T.lap("layout: incidence + stencils");
        if (given) {
            c->colour = *given;
            c->ncol = 0;
            for (int32_t k : c->colour) c->ncol = std::max(c->ncol, k + 1);
        } else {
            c->colour.assign((size_t)nv, 0);
            pbng_status st = colour_greedy(c, vs_off, vs);
            if (st != PBNG_OK) return st;
        }
        // ---- which vertices this context holds (domain decomposition; one rank = everything) ----------
        // need[v] = ranks that hold v: a rank holds every vertex of a stencil touching one of its free
        // vertices, and the vertices of the tets / constraints whose energy it evaluates (owner of the
        // first vertex).  The colouring above is global, identical on every rank.
        const int32_t me = c->rank, nranks = c->n_ranks;
        std::vector<int32_t> own = c->owner.empty() ? std::vector<int32_t>((size_t)nv, 0) : c->owner;
        std::vector<uint64_t> need((size_t)nv, 0ull);
        auto bit = [](int32_t r) { return 1ull << r; };
        for (int64_t e = 0; e < nt; ++e) {
            const int32_t *t = c->tets.data() + 4 * e;
            uint64_t m = bit(own[t[0]]);
            for (int a = 0; a < 4; ++a)
                if (!is_pinned[t[a]]) m |= bit(own[t[a]]);
            for (int a = 0; a < 4; ++a) need[t[a]] |= m;
        }
        for (int64_t q = 0; q < nwc; ++q) {
            uint64_t m = bit(own[c->wc[q].idx0[0]]);
            for (int32_t v : cnodes[q])
                if (!is_pinned[v]) m |= bit(own[v]);
            for (int32_t v : cnodes[q]) need[v] |= m;
        }
        for (int64_t v = 0; v < nv; ++v) {
            if (!is_pinned[v]) need[v] |= bit(own[v]);
            else if (nranks == 1) need[v] |= 1ull;
        }
        auto held = [&](int64_t v) { return ((need[v] >> me) & 1ull) != 0; };
        // an owned free vertex another rank holds is sent after its colour pass: laid out first in its
        // colour so that its part of the pass can run before the rest (dd.py overlaps the exchange)
        auto is_send = [&](int64_t v) { return !is_pinned[v] && own[v] == me && (need[v] & ~bit(me)) != 0ull; };
        // permutation: owned free vertices colour-major | ghost free vertices | held pinned vertices
        c->col_vbegin.assign(c->ncol + 1, 0);
        c->col_nfree.assign(c->ncol, 0);
        c->gcol_nfree.assign(c->ncol, 0);
        for (int64_t v = 0; v < nv; ++v)
            if (!is_pinned[v]) {
                c->gcol_nfree[c->colour[v]]++;
                if (own[v] == me) c->col_nfree[c->colour[v]]++;
            }
        for (int32_t k = 0; k < c->ncol; ++k) c->col_vbegin[k + 1] = c->col_vbegin[k] + c->col_nfree[k];
        c->n_free = c->col_vbegin[c->ncol];
        c->col_nsend.assign(c->ncol, 0);
        for (int64_t v = 0; v < nv; ++v)
            if (is_send(v)) c->col_nsend[c->colour[v]]++;
        c->orig2int.assign((size_t)nv, -1);
        c->int2orig.assign((size_t)c->n_free, 0);
        {
            std::vector<int32_t> fill(c->col_vbegin.begin(), c->col_vbegin.end() - 1);
            for (int pass = 0; pass < 2; ++pass)  // halo-send vertices first within each colour
                for (int64_t v = 0; v < nv; ++v)
                    if (!is_pinned[v] && own[v] == me && is_send(v) == (pass == 0)) {
                        const int32_t i = fill[c->colour[v]]++;
                        c->orig2int[v] = i;
                        c->int2orig[i] = (int32_t)v;
                    }
            for (int64_t v = 0; v < nv; ++v)
                if (!is_pinned[v] && own[v] != me && held(v)) {
                    c->orig2int[v] = (int32_t)c->int2orig.size();
                    c->int2orig.push_back((int32_t)v);
                }
            c->n_local_free = (int64_t)c->int2orig.size();
            c->local_pinned.clear();
            for (size_t k = 0; k < c->pinned.size(); ++k)
                if (held(c->pinned[k])) {
                    c->orig2int[c->pinned[k]] = (int32_t)c->int2orig.size();
                    c->int2orig.push_back(c->pinned[k]);
                    c->local_pinned.push_back((int32_t)k);
                }
            c->n_local = (int64_t)c->int2orig.size();
        }
        // energy ownership: tets and constraints by the owner of their first vertex
        c->tet_local.clear();
        for (int64_t e = 0; e < nt; ++e)
            if (own[c->tets[4 * e]] == me) c->tet_local.push_back((int32_t)e);
        c->cons_local.clear();
        for (int64_t q = 0; q < nwc; ++q)
            if (own[c->wc[q].idx0[0]] == me) c->cons_local.push_back((int32_t)q);
        c->n_cons_owned = (int64_t)c->cons_local.size();
        for (int64_t q = 0; q < nwc; ++q) {
            if (own[c->wc[q].idx0[0]] == me) continue;
            bool touches = false;
            for (int32_t v : cnodes[q]) touches |= (!is_pinned[v] && own[v] == me);
            if (touches) c->cons_local.push_back((int32_t)q);
        }
        // halo plan: after colour k, rank `me` sends its owned colour-k vertices held by peer p and
        // receives the colour-k vertices of p that it holds; both lists ascending in original index
        c->halo_send_off.assign((size_t)c->ncol * nranks + 1, 0);
        c->halo_recv_off.assign((size_t)c->ncol * nranks + 1, 0);
        c->halo_send_orig.clear();
        c->halo_recv_orig.clear();
        if (nranks > 1) {
            std::vector<std::vector<int32_t>> snd((size_t)c->ncol * nranks), rcv((size_t)c->ncol * nranks);
            for (int64_t v = 0; v < nv; ++v) {
                if (is_pinned[v]) continue;
                const int32_t k = c->colour[v];
                if (own[v] == me) {
                    for (int32_t p = 0; p < nranks; ++p)
                        if (p != me && ((need[v] >> p) & 1ull)) snd[(size_t)k * nranks + p].push_back((int32_t)v);
                } else if (held(v)) {
                    rcv[(size_t)k * nranks + own[v]].push_back((int32_t)v);
                }
            }
            for (size_t s = 0; s < snd.size(); ++s) {
                c->halo_send_off[s + 1] = c->halo_send_off[s] + (int64_t)snd[s].size();
                c->halo_recv_off[s + 1] = c->halo_recv_off[s] + (int64_t)rcv[s].size();
                c->halo_send_orig.insert(c->halo_send_orig.end(), snd[s].begin(), snd[s].end());
                c->halo_recv_orig.insert(c->halo_recv_orig.end(), rcv[s].begin(), rcv[s].end());
            }
        }
        // Within a colour the update order is free (same-coloured vertices share no stencil, PAPER.md:
        // 697-705), so each colour's free vertices are laid out along a Morton curve of their rest
        // positions: a warp's 32 vertices are spatially compact and their neighbour gathers share cache
        // lines.  Results are unchanged bit for bit (each vertex's own summation order is fixed).
        if (spatial_order()) {
            double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
            for (int64_t v = 0; v < nv; ++v)
                for (int a = 0; a < 3; ++a) {
                    lo[a] = std::min(lo[a], c->X[3 * v + a]);
                    hi[a] = std::max(hi[a], c->X[3 * v + a]);
                }
            double ext = 0;
            for (int a = 0; a < 3; ++a) ext = std::max(ext, hi[a] - lo[a]);
            const double scale = ext > 0 ? (double)((1u << 21) - 1) / ext : 0.0;
            std::vector<uint64_t> key((size_t)nv);
            for (int64_t v = 0; v < nv; ++v) {
                uint64_t q[3];
                for (int a = 0; a < 3; ++a) q[a] = (uint64_t)((c->X[3 * v + a] - lo[a]) * scale);
                key[v] = morton3(q[0], q[1], q[2]);
            }
            for (int32_t col = 0; col < c->ncol; ++col) {  // each part (halo-send | rest) sorted on its own
                int32_t *b = c->int2orig.data() + c->col_vbegin[col];
                const int32_t ns = c->col_nsend[col];
                std::stable_sort(b, b + ns, [&](int32_t x, int32_t y) { return key[x] < key[y]; });
                std::stable_sort(b + ns, b + c->col_nfree[col], [&](int32_t x, int32_t y) { return key[x] < key[y]; });
                for (int32_t q = 0; q < c->col_nfree[col]; ++q) c->orig2int[b[q]] = c->col_vbegin[col] + q;
            }
        }
        c->h_halo_send.resize(c->halo_send_orig.size());
        c->h_halo_recv.resize(c->halo_recv_orig.size());
        for (size_t q = 0; q < c->halo_send_orig.size(); ++q) c->h_halo_send[q] = c->orig2int[c->halo_send_orig[q]];
        for (size_t q = 0; q < c->halo_recv_orig.size(); ++q) c->h_halo_recv[q] = c->orig2int[c->halo_recv_orig[q]];
        T.lap("layout: colouring + ownership + order");
        if (c->dtype == DT_F64) build_layout<double>(c, vt_off, vt);
        else build_layout<float>(c, vt_off, vt);
        T.lap("layout: records");
        build_pipeline(c, vt_off, vt);
        T.lap("layout: pipeline dependencies");
        build_surface(c);
        T.lap("layout: surface");
        plan_workspace(c);
    } catch (const std::bad_alloc &) {
        return fail(PBNG_E_OUT_OF_MEMORY, "color: host allocation");
    }
    c->colored = true;
    c->bound = false;
    c->positions_set = false;
    return PBNG_OK;
}

pbng_status pbng_color(pbng_ctx *c, int32_t *colour_out, int32_t *n_colours_out) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (!c->has_material || !c->has_constraints)
        return fail(PBNG_E_BAD_ORDER, "color: set_material and set_constraints must come first");
    pbng_status st = colour_and_layout(c, nullptr);
    if (st != PBNG_OK) return st;
    if (colour_out) std::memcpy(colour_out, c->colour.data(), (size_t)c->nv * 4);
    if (n_colours_out) *n_colours_out = c->ncol;
    return PBNG_OK;
}

pbng_status pbng_color_given(pbng_ctx *c, const int32_t *colours, int32_t *n_colours_out, int64_t *bad_index) {
    if (bad_index) *bad_index = -1;
    if (!c || !colours) return fail(PBNG_E_INVALID_ARGUMENT, "color_given: null argument");
    if (!c->has_material || !c->has_constraints)
        return fail(PBNG_E_BAD_ORDER, "color_given: set_material and set_constraints must come first");
    // a node colouring in the sense of PAPER.md:702: nodes of one colour share no element and no weak constraint
    for (int64_t v = 0; v < c->nv; ++v)
        if (colours[v] < 0 || colours[v] >= 65536) {
            if (bad_index) *bad_index = v;
            return fail(PBNG_E_INVALID_ARGUMENT, "color_given: colour of vertex " + std::to_string(v) + " outside [0, 65536)");
        }
    for (int64_t e = 0; e < c->nt; ++e) {
        const int32_t *t = c->tets.data() + 4 * e;
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b)
                if (t[a] != t[b] && colours[t[a]] == colours[t[b]]) {
                    if (bad_index) *bad_index = e;
                    return fail(PBNG_E_INVALID_ARGUMENT, "color_given: two vertices of tet " + std::to_string(e) + " share a colour");
                }
    }
    for (size_t q = 0; q < c->wc.size(); ++q) {
        const pbng_weak_constraint &w = c->wc[q];
        std::vector<int32_t> nodes;
        for (int a = 0; a < w.n0; ++a) nodes.push_back(w.idx0[a]);
        for (int a = 0; a < w.n1; ++a) nodes.push_back(w.idx1[a]);
        std::sort(nodes.begin(), nodes.end());
        nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
        for (size_t a = 0; a < nodes.size(); ++a)
            for (size_t b = a + 1; b < nodes.size(); ++b)
                if (colours[nodes[a]] == colours[nodes[b]]) {
                    if (bad_index) *bad_index = c->nt + (int64_t)q;
                    return fail(PBNG_E_INVALID_ARGUMENT, "color_given: two nodes of weak constraint " + std::to_string(q) + " share a colour");
                }
    }
    const std::vector<int32_t> given(colours, colours + c->nv);
    pbng_status st = colour_and_layout(c, &given);
    if (st != PBNG_OK) return st;
    if (n_colours_out) *n_colours_out = c->ncol;
    return PBNG_OK;
}

pbng_status pbng_workspace_bytes(pbng_ctx *c, uint64_t *bytes) {
    if (!c || !bytes) return fail(PBNG_E_INVALID_ARGUMENT, "null argument");
    if (!c->colored) return fail(PBNG_E_NOT_COLORED, "workspace_bytes: call pbng_color first");
    *bytes = c->ws_need;
    return PBNG_OK;
}

}  // extern "C"

// Upload the host images into the workspace and point the layout at it.  fresh = false (re-layout of
// pbng_update_constraints): the position, inertial-target and staging regions, which sit first at offsets
// the re-layout does not change, are left alone, and the iterate state is kept.
static pbng_status bind_layout(pbng_ctx *c, void *dptr, uint64_t bytes, bool fresh) {
    DevGuard g(c->device);
    char *base = static_cast<char *>(dptr);
    auto at = [&](const Region &r) { return static_cast<void *>(base + r.off); };
    Layout L;
    L.n_vertices = c->n_local;
    L.n_slots = c->n_slots;
    L.rec_id = static_cast<const int4 *>(at(c->r_rec_id));
    L.path0 = static_cast<const int2 *>(at(c->r_path0));
    L.rec_a = at(c->r_rec_a);
    L.rec_b = at(c->r_rec_b);
    L.rec_c = at(c->r_rec_c);
    L.rest = c->rest_rec ? at(c->r_rest) : nullptr;
    L.path_mode = c->prob.path_mode;
    L.n_tab = c->prob.path_mode == 3 ? (int32_t)c->n_tab : 0;
    L.chunk_off = static_cast<const int64_t *>(at(c->r_chunk_off));
    L.chunk_v = static_cast<const int2 *>(at(c->r_chunk_v));
    L.deg = static_cast<const int32_t *>(at(c->r_deg));
    L.fext = c->prob.has_fext ? at(c->r_fext) : nullptr;
    L.wc_off = static_cast<const int32_t *>(at(c->r_wc_off));
    L.wc_cid = static_cast<const int32_t *>(at(c->r_wc_cid));
    L.wc_d = at(c->r_wc_d);
    L.c_n = static_cast<const int32_t *>(at(c->r_c_n));
    L.c_node = static_cast<const int32_t *>(at(c->r_c_node));
    L.c_w = at(c->r_c_w);
    L.c_anchor = at(c->r_c_anchor);
    L.c_K = at(c->r_c_K);
    L.tet_id = static_cast<const int4 *>(at(c->r_tet_id));
    L.tet_a = at(c->r_tet_a);
    L.tet_b = at(c->r_tet_b);
    L.tet_c = at(c->r_tet_c);
    L.int2orig = static_cast<const int32_t *>(at(c->r_int2orig));
    L.targets = at(c->r_targets);
    for (int k = 0; k < 3; ++k) L.xbuf[k] = at(c->r_x[k]);
    L.stage = at(c->r_stage);
    c->stage2 = at(c->r_stage2);
    L.part_e = static_cast<double *>(at(c->r_part_e));
    L.part_r = static_cast<double *>(at(c->r_part_r));
    L.results = static_cast<double *>(at(c->r_results));
    L.flag = static_cast<int32_t *>(at(c->r_flag));
    L.mass = at(c->r_mass);
    L.xtilde = at(c->r_xt);
    L.halo_send = static_cast<const int32_t *>(at(c->r_halo_send));
    L.halo_recv = static_cast<const int32_t *>(at(c->r_halo_recv));
    L.surf = static_cast<const int4 *>(at(c->r_surf));
    L.sv = static_cast<const int2 *>(at(c->r_sv));
    L.c_head = static_cast<int32_t *>(at(c->r_chead));
    L.c_next = static_cast<int2 *>(at(c->r_cnext));
    L.c_res = static_cast<ContactHit *>(at(c->r_cres));
    L.c_scal = static_cast<uint32_t *>(at(c->r_cscal));
    L.dep_off = static_cast<const int32_t *>(at(c->r_dep_off));
    L.deps = static_cast<const int32_t *>(at(c->r_deps));
    L.pipe_counter = static_cast<uint64_t *>(at(c->r_pipe));
    L.pipe_flags = reinterpret_cast<int32_t *>(static_cast<char *>(at(c->r_pipe)) + 8);
    auto up = [&](const Region &r, const void *src, size_t n) -> cudaError_t {
        if (n == 0) return cudaSuccess;
        return cudaMemcpyAsync(base + r.off, src, n, cudaMemcpyHostToDevice, c->stream);
    };
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
    if (c->path_rec) chk(up(c->r_rec_id, c->h_rec_id2.data(), c->h_rec_id2.size() * 8));
    else chk(up(c->r_rec_id, c->h_rec_id.data(), c->h_rec_id.size() * 16));
    chk(up(c->r_path0, c->h_path0.data(), c->h_path0.size() * 8));
    chk(up(c->r_rec_a, c->h_rec_a.data(), c->h_rec_a.size()));
    chk(up(c->r_rest, c->h_rest.data(), c->h_rest.size()));
    chk(up(c->r_rec_b, c->h_rec_b.data(), c->h_rec_b.size()));
    chk(up(c->r_rec_c, c->h_rec_c.data(), c->h_rec_c.size()));
    chk(up(c->r_chunk_off, c->h_chunk_off.data(), c->h_chunk_off.size() * 8));
    chk(up(c->r_chunk_v, c->h_chunk_v.data(), c->h_chunk_v.size() * 8));
    chk(up(c->r_deg, c->h_deg.data(), c->h_deg.size() * 4));
    chk(up(c->r_fext, c->h_fext.data(), c->h_fext.size()));
    chk(up(c->r_wc_off, c->h_wc_off.data(), c->h_wc_off.size() * 4));
    chk(up(c->r_wc_cid, c->h_wc_cid.data(), c->h_wc_cid.size() * 4));
    chk(up(c->r_wc_d, c->h_wc_d.data(), c->h_wc_d.size()));
    chk(up(c->r_c_n, c->h_c_n.data(), c->h_c_n.size() * 4));
    chk(up(c->r_c_node, c->h_c_node.data(), c->h_c_node.size() * 4));
    chk(up(c->r_c_w, c->h_c_w.data(), c->h_c_w.size()));
    chk(up(c->r_c_anchor, c->h_c_anchor.data(), c->h_c_anchor.size()));
    chk(up(c->r_c_K, c->h_c_K.data(), c->h_c_K.size()));
    chk(up(c->r_tet_id, c->h_tet_id.data(), c->h_tet_id.size() * 16));
    chk(up(c->r_tet_a, c->h_tet_a.data(), c->h_tet_a.size()));
    chk(up(c->r_tet_b, c->h_tet_b.data(), c->h_tet_b.size()));
    chk(up(c->r_tet_c, c->h_tet_c.data(), c->h_tet_c.size()));
    chk(up(c->r_int2orig, c->int2orig.data(), c->int2orig.size() * 4));
    chk(up(c->r_mass, c->h_mass.data(), c->h_mass.size()));
    chk(up(c->r_halo_send, c->h_halo_send.data(), c->h_halo_send.size() * 4));
    chk(up(c->r_halo_recv, c->h_halo_recv.data(), c->h_halo_recv.size() * 4));
    chk(up(c->r_targets, c->h_targets.data(), c->h_targets.size()));
    chk(up(c->r_surf, c->h_surf.data(), c->h_surf.size() * 16));
    chk(up(c->r_sv, c->h_sv.data(), c->h_sv.size() * 8));
    chk(up(c->r_dep_off, c->h_dep_off.data(), c->h_dep_off.size() * 4));
    chk(up(c->r_deps, c->h_deps.data(), c->h_deps.size() * 4));
    if (fresh) {
        chk(cudaMemsetAsync(base + c->r_flag.off, 0, 4, c->stream));
        // position buffers start at zero: padding rows / lanes (x_stride, sample groups) are then finite
        for (int k = 0; k < 3; ++k) chk(cudaMemsetAsync(base + c->r_x[k].off, 0, c->r_x[k].bytes, c->stream));
        chk(cudaMemsetAsync(base + c->r_xt.off, 0, c->r_xt.bytes, c->stream));
    }
    chk(cudaStreamSynchronize(c->stream));
    if (e != cudaSuccess) return cuda_fail(e, "bind_workspace");
    drop_dd_graph(c);  // a captured iterate block holds the old layout and buffers
    c->layout_gen += 1;
    c->ws = dptr;
    c->ws_bytes = bytes;
    c->L = L;
    c->bound = true;
    if (fresh) c->positions_set = false;
    if (c->l2_persist && fresh) return apply_l2_persistence(c, 1);  // the position buffers may have moved
    return PBNG_OK;
}

extern "C" {

pbng_status pbng_bind_workspace(pbng_ctx *c, void *dptr, uint64_t bytes) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->colored) return fail(PBNG_E_NOT_COLORED, "bind_workspace: call pbng_color first");
    if (!dptr || (reinterpret_cast<uintptr_t>(dptr) & 255u) != 0)
        return fail(PBNG_E_INVALID_ARGUMENT, "bind_workspace: pointer must be non-null and 256-byte aligned");
    if (bytes < c->ws_need) return fail(PBNG_E_OUT_OF_MEMORY, "bind_workspace: workspace smaller than pbng_workspace_bytes");
    return bind_layout(c, dptr, bytes, true);
}

pbng_status pbng_set_positions(pbng_ctx *c, const void *x) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->bound) return fail(PBNG_E_BAD_ORDER, "set_positions: bind a workspace first");
    if (!x) return fail(PBNG_E_INVALID_ARGUMENT, "set_positions: null pointer");
    DevGuard g(c->device);
    const size_t n = (size_t)c->nb * (size_t)c->nv * 3 * c->real_size();
    PBNG_CUDA(cudaMemcpyAsync(c->L.stage, x, n, cudaMemcpyDefault, c->stream), "set_positions: copy");
    PBNG_CUDA(cudaMemsetAsync(c->L.flag, 0, 4, c->stream), "set_positions: flag");
    PBNG_CUDA(launch_set_positions(c->prob, c->L, 3, c->stream), "set_positions: kernel");
    c->launches += 1;
    c->work = 0;
    c->out = 1;
    c->hist = 2;
    c->l = 0;
    c->hist_valid = true;
    c->positions_set = true;
    c->cur_accel = -1;
    return PBNG_OK;
}

pbng_status pbng_set_inertia(pbng_ctx *c, double dt, const void *xtilde) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->bound) return fail(PBNG_E_BAD_ORDER, "set_inertia: bind a workspace first");
    if (!(dt >= 0.0) || !std::isfinite(dt)) return fail(PBNG_E_INVALID_ARGUMENT, "set_inertia: dt must be >= 0");
    if (dt == 0.0) {
        c->prob.inv_dt2 = 0.0;
        return PBNG_OK;
    }
    if (!(c->density > 0.0)) return fail(PBNG_E_INVALID_ARGUMENT, "set_inertia: backward Euler needs density > 0");
    if (!xtilde) return fail(PBNG_E_INVALID_ARGUMENT, "set_inertia: null xtilde");
    DevGuard g(c->device);
    const size_t n = (size_t)c->nb * (size_t)c->nv * 3 * c->real_size();
    PBNG_CUDA(cudaMemcpyAsync(c->L.stage, xtilde, n, cudaMemcpyDefault, c->stream), "set_inertia: copy");
    PBNG_CUDA(launch_set_positions(c->prob, c->L, -1, c->stream), "set_inertia: kernel");
    c->launches += 1;
    c->prob.inv_dt2 = 1.0 / (dt * dt);
    return PBNG_OK;
}

pbng_status pbng_get_positions(pbng_ctx *c, void *x_out) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->positions_set) return fail(PBNG_E_BAD_ORDER, "get_positions: set_positions first");
    if (!x_out) return fail(PBNG_E_INVALID_ARGUMENT, "get_positions: null pointer");
    DevGuard g(c->device);
    PBNG_CUDA(launch_get_positions(c->prob, c->L, c->work, c->stream), "get_positions: kernel");
    c->launches += 1;
    const size_t n = (size_t)c->nb * (size_t)c->nv * 3 * c->real_size();
    PBNG_CUDA(cudaMemcpyAsync(x_out, c->L.stage, n, cudaMemcpyDefault, c->stream), "get_positions: copy");
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, x_out) != cudaSuccess) {
        cudaGetLastError();
        attr.type = cudaMemoryTypeUnregistered;
    }
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
        PBNG_CUDA(cudaStreamSynchronize(c->stream), "get_positions: synchronize");
    return PBNG_OK;
}

pbng_status pbng_iterate(pbng_ctx *c, int32_t n_iterations, pbng_accel accel, double omega, double rho, double gamma) {
    pbng_status st = check_iterate(c, accel, omega, rho, gamma, "iterate");
    if (st != PBNG_OK) return st;
    if (n_iterations < 0) return fail(PBNG_E_INVALID_ARGUMENT, "iterate: negative iteration count");
    if (c->cur_accel >= 0) return fail(PBNG_E_BAD_ORDER, "iterate: an iteration started by pbng_sweep_colour is open");
    DevGuard g(c->device);
    std::pair<cudaEvent_t, cudaEvent_t> span;
    const bool span_prof = c->profiling == 2 && n_iterations > 0;
    int64_t span_launches = 0;
    if (span_prof) {
        PBNG_CUDA(get_event_pair(c, span), "iterate: profiling events");
        PBNG_CUDA(cudaEventRecord(span.first, c->stream), "iterate: event");
    }
    if (c->n_ranks > 1) {
        // decomposed: the per-colour halo exchange runs inside the library (pbng_partition's NCCL
        // communicator); without one the caller drives the colours (pbng_sweep_colour_part + halo calls)
        if (!c->comm)
            return fail(PBNG_E_BAD_ORDER, "iterate: decomposed context without a transport (pbng_partition with an "
                                          "NCCL id, pbng_group_iterate, or the colour-by-colour calls)");
        PBNG_CUDA(ensure_dd_streams(c), "iterate: side stream");
        Exchange X;
        X.ranks = {c};
        if (c->peer.enabled) {
            if (peer_stale(c))
                return fail(PBNG_E_BAD_ORDER, "iterate: the layout or workspace changed since pbng_enable_peer_halo; "
                                              "call it again on every rank");
            X.peer = true;
        }
        int64_t sweeps = 0;
        st = dd_run(c, X, c->stream, c->dd_side, c->dd_cap, c->dd_ev_a, c->dd_ev_b, n_iterations, accel, omega, rho,
                    gamma, &sweeps, "iterate: decomposed iterations");
        if (st != PBNG_OK) return st;
        span_launches += sweeps;
    } else if (b2_window_schedule(c)) {
        // batched fp32 NH (sh 6): windowed persistent launches, one per kPipeMaxIter iterations
        for (int32_t it = 0; it < n_iterations; it += kPipeMaxIter) {
            B2Window W;
            W.n_iter = std::min<int32_t>(kPipeMaxIter, n_iterations - it);
            W.ncol = c->ncol;
            W.window = b2_window_size(c);
            W.work = c->work;
            W.out = c->out;
            W.hist = c->hist;
            W.gamma = accel == PBNG_ACCEL_CHEBYSHEV ? gamma : 1.0;
            for (int j = 0; j < W.n_iter; ++j)
                W.omega[j] = accel == PBNG_ACCEL_SOR ? omega
                             : accel == PBNG_ACCEL_CHEBYSHEV ? chebyshev_weight(c->l + j + 1, rho) : 1.0;
            constexpr int WPB = kSweepBlock / 32 * kB2WinVpw;  // vertices per item
            W.blk_off[0] = 0;
            for (int32_t col = 0; col < c->ncol; ++col) {
                W.v_begin[col] = c->col_vbegin[col];
                W.n_v[col] = c->col_nfree[col];
                W.chunk_begin[col] = c->col_chunk[col];
                W.blk_off[col + 1] = W.blk_off[col] + (c->col_nfree[col] + WPB - 1) / WPB;
            }
            // an empty colour has no items: each colour waits for the previous colour WITH vertices (so the
            // chain of waits still orders every colour pass of a group pair)
            for (int32_t col = 0; col < c->ncol; ++col) {
                int32_t pc = col;
                for (int k = 1; k <= c->ncol; ++k) {
                    const int32_t q = (col - k + c->ncol) % c->ncol;
                    if (W.blk_off[q + 1] > W.blk_off[q]) {
                        pc = q;
                        break;
                    }
                }
                W.prev[col] = pc;
            }
            const size_t n_gp = (size_t)((c->nb + 63) / 64);
            PBNG_CUDA(cudaMemsetAsync(c->L.pipe_counter, 0, 8 + n_gp * (size_t)c->ncol * 4, c->stream), "iterate: window reset");
            PBNG_CUDA(timed_launch(c, [&] { return launch_b2_window(c->prob, c->L, W, (int)accel, c->stream); }),
                      "iterate: windowed batched sweep");
            c->launches += 1;
            span_launches += 1;
            for (int j = 0; j < W.n_iter; ++j) end_iteration_impl(c, accel);
        }
    } else if (effective_schedule(c) == 2) {
        // pipelined: one persistent launch per kPipeMaxIter iterations, no barrier between colours
        for (int32_t it = 0; it < n_iterations; it += kPipeMaxIter) {
            PipeLaunch P;
            P.n_iter = std::min<int32_t>(kPipeMaxIter, n_iterations - it);
            P.accel = accel;
            P.work = c->work;
            P.out = c->out;
            P.hist = c->hist;
            P.split = problem_split(c);
            P.gamma = accel == PBNG_ACCEL_CHEBYSHEV ? gamma : 1.0;
            for (int j = 0; j < P.n_iter; ++j)
                P.omega[j] = accel == PBNG_ACCEL_SOR ? omega
                             : accel == PBNG_ACCEL_CHEBYSHEV ? chebyshev_weight(c->l + j + 1, rho) : 1.0;
            PBNG_CUDA(cudaMemsetAsync(c->L.pipe_counter, 0, c->r_pipe.bytes, c->stream), "iterate: pipeline reset");
            PBNG_CUDA(timed_launch(c, [&] { return launch_sweep_pipe(c->prob, c->L, P, c->stream); }), "iterate: pipelined sweep");
            c->launches += 1;
            span_launches += 1;
            for (int j = 0; j < P.n_iter; ++j) end_iteration_impl(c, accel);
        }
    } else {
        for (int32_t it = 0; it < n_iterations; ++it) {
            for (int32_t col = 0; col < c->ncol; ++col) {
                PBNG_CUDA(sweep_colour_impl(c, col, accel, omega, rho, gamma, &span_launches), "iterate: sweep kernel");
            }
            end_iteration_impl(c, accel);
        }
    }
    if (span_prof) {
        PBNG_CUDA(cudaEventRecord(span.second, c->stream), "iterate: event");
        c->ev_used.push_back(span);
        c->ev_launches.push_back(span_launches);
    }
    return PBNG_OK;
}

pbng_status pbng_sweep_colour(pbng_ctx *c, int32_t colour, pbng_accel accel, double omega, double rho, double gamma) {
    pbng_status st = check_iterate(c, accel, omega, rho, gamma, "sweep_colour");
    if (st != PBNG_OK) return st;
    if (colour < 0 || colour >= c->ncol) return fail(PBNG_E_INVALID_ARGUMENT, "sweep_colour: colour out of range");
    if (c->cur_accel >= 0 && c->cur_accel != (int)accel)
        return fail(PBNG_E_BAD_ORDER, "sweep_colour: acceleration changed within an iteration");
    DevGuard g(c->device);
    int64_t n = 0;
    PBNG_CUDA(sweep_colour_impl(c, colour, accel, omega, rho, gamma, &n), "sweep_colour: sweep kernel");
    c->cur_accel = (int)accel;
    return PBNG_OK;
}

pbng_status pbng_sweep_colour_part(pbng_ctx *c, int32_t colour, int32_t part, pbng_accel accel, double omega,
                                   double rho, double gamma) {
    pbng_status st = check_iterate(c, accel, omega, rho, gamma, "sweep_colour_part");
    if (st != PBNG_OK) return st;
    if (colour < 0 || colour >= c->ncol) return fail(PBNG_E_INVALID_ARGUMENT, "sweep_colour_part: colour out of range");
    if (part < 0 || part > 2) return fail(PBNG_E_INVALID_ARGUMENT, "sweep_colour_part: part must be 0, 1 or 2");
    if (c->cur_accel >= 0 && c->cur_accel != (int)accel)
        return fail(PBNG_E_BAD_ORDER, "sweep_colour_part: acceleration changed within an iteration");
    DevGuard g(c->device);
    int64_t n = 0;
    PBNG_CUDA(sweep_colour_impl(c, colour, accel, omega, rho, gamma, &n, part), "sweep_colour_part: sweep kernel");
    c->cur_accel = (int)accel;
    return PBNG_OK;
}

pbng_status pbng_set_stream(pbng_ctx *c, uintptr_t cuda_stream) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    const cudaStream_t s = reinterpret_cast<cudaStream_t>(cuda_stream);
    if (s == c->stream) return PBNG_OK;
    c->stream = s;
    // the L2 window belongs to the stream the context issues on: move it (and never leave it behind)
    if (c->l2_applied) return apply_l2_persistence(c, 1);
    return PBNG_OK;
}

pbng_status pbng_end_iteration(pbng_ctx *c, pbng_accel accel) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (c->cur_accel < 0 || c->cur_accel != (int)accel)
        return fail(PBNG_E_BAD_ORDER, "end_iteration: no colour pass of this acceleration is open");
    end_iteration_impl(c, accel);
    return PBNG_OK;
}

pbng_status pbng_set_partition(pbng_ctx *c, const int32_t *owner, int32_t rank, int32_t n_ranks) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (n_ranks < 1 || n_ranks > 64 || rank < 0 || rank >= n_ranks)
        return fail(PBNG_E_INVALID_ARGUMENT, "set_partition: need 1 <= n_ranks <= 64 and 0 <= rank < n_ranks");
    if (n_ranks > 1 && !owner) return fail(PBNG_E_INVALID_ARGUMENT, "set_partition: owner is null");
    try {
        std::vector<int32_t> o;
        if (n_ranks > 1) {
            o.assign(owner, owner + c->nv);
            for (int64_t v = 0; v < c->nv; ++v)
                if (o[v] < 0 || o[v] >= n_ranks)
                    return fail(PBNG_E_INDEX_OUT_OF_RANGE, "set_partition: owner rank out of range at vertex " + std::to_string(v));
        }
        c->owner.swap(o);
    } catch (const std::bad_alloc &) {
        return fail(PBNG_E_OUT_OF_MEMORY, "set_partition: host allocation");
    }
    c->rank = rank;
    c->n_ranks = n_ranks;
    c->invalidate_colouring();
    return PBNG_OK;
}

static pbng_status halo_segment(pbng_ctx *c, int32_t colour, int32_t peer, size_t *seg, const char *who) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (!c->colored) return fail(PBNG_E_NOT_COLORED, std::string(who) + ": call pbng_color first");
    if (colour < 0 || colour >= c->ncol || peer < 0 || peer >= c->n_ranks)
        return fail(PBNG_E_INVALID_ARGUMENT, std::string(who) + ": colour or peer out of range");
    *seg = (size_t)colour * (size_t)c->n_ranks + (size_t)peer;
    return PBNG_OK;
}

pbng_status pbng_halo_counts(pbng_ctx *c, int32_t colour, int32_t peer, int64_t *n_send, int64_t *n_recv) {
    size_t seg = 0;
    pbng_status st = halo_segment(c, colour, peer, &seg, "halo_counts");
    if (st != PBNG_OK) return st;
    const bool dd = c->n_ranks > 1;
    if (n_send) *n_send = dd ? c->halo_send_off[seg + 1] - c->halo_send_off[seg] : 0;
    if (n_recv) *n_recv = dd ? c->halo_recv_off[seg + 1] - c->halo_recv_off[seg] : 0;
    return PBNG_OK;
}

pbng_status pbng_halo_vertices(pbng_ctx *c, int32_t colour, int32_t peer, int32_t *send_vertices, int32_t *recv_vertices) {
    size_t seg = 0;
    pbng_status st = halo_segment(c, colour, peer, &seg, "halo_vertices");
    if (st != PBNG_OK) return st;
    if (c->n_ranks == 1) return PBNG_OK;
    if (send_vertices)
        std::copy(c->halo_send_orig.begin() + c->halo_send_off[seg], c->halo_send_orig.begin() + c->halo_send_off[seg + 1],
                  send_vertices);
    if (recv_vertices)
        std::copy(c->halo_recv_orig.begin() + c->halo_recv_off[seg], c->halo_recv_orig.begin() + c->halo_recv_off[seg + 1],
                  recv_vertices);
    return PBNG_OK;
}

static pbng_status halo_io(pbng_ctx *c, int32_t colour, int32_t peer, int32_t n_fields, const void *buf, bool pack) {
    const char *who = pack ? "halo_pack" : "halo_unpack";
    size_t seg = 0;
    pbng_status st = halo_segment(c, colour, peer, &seg, who);
    if (st != PBNG_OK) return st;
    st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->positions_set) return fail(PBNG_E_BAD_ORDER, std::string(who) + ": set_positions first");
    if (n_fields != 1 && n_fields != 3) return fail(PBNG_E_INVALID_ARGUMENT, std::string(who) + ": n_fields must be 1 or 3");
    if (c->n_ranks == 1) return PBNG_OK;
    const int64_t off = pack ? c->halo_send_off[seg] : c->halo_recv_off[seg];
    const int64_t n = (pack ? c->halo_send_off[seg + 1] : c->halo_recv_off[seg + 1]) - off;
    if (n == 0) return PBNG_OK;
    if (!buf) return fail(PBNG_E_INVALID_ARGUMENT, std::string(who) + ": null buffer");
    DevGuard g(c->device);
    const int bufs[3] = {c->work, c->out, c->hist};
    cudaError_t e = pack ? launch_halo_pack(c->prob, c->L, c->L.halo_send + off, n, n_fields, bufs, const_cast<void *>(buf), c->stream)
                         : launch_halo_unpack(c->prob, c->L, c->L.halo_recv + off, n, n_fields, bufs, buf, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, who);
    c->launches += 1;
    return PBNG_OK;
}

pbng_status pbng_halo_pack(pbng_ctx *c, int32_t colour, int32_t peer, int32_t n_fields, void *device_buffer) {
    return halo_io(c, colour, peer, n_fields, device_buffer, true);
}

pbng_status pbng_halo_unpack(pbng_ctx *c, int32_t colour, int32_t peer, int32_t n_fields, const void *device_buffer) {
    return halo_io(c, colour, peer, n_fields, device_buffer, false);
}

pbng_status pbng_synchronize(pbng_ctx *c) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    DevGuard g(c->device);
    PBNG_CUDA(cudaStreamSynchronize(c->stream), "synchronize");
    if (c->bound) {
        int32_t flag = 0;
        PBNG_CUDA(cudaMemcpy(&flag, c->L.flag, 4, cudaMemcpyDeviceToHost), "synchronize: flag");
        if (flag & 2) return fail(PBNG_E_CUDA, "peer halo: a neighbour rank's signal did not arrive in time");
        if (flag) return fail(PBNG_E_NONFINITE, "a non-finite position was produced");
    }
    return PBNG_OK;
}

pbng_status pbng_energy_residual(pbng_ctx *c, double *energy_out, double *residual_out) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->positions_set) return fail(PBNG_E_BAD_ORDER, "energy_residual: set_positions first");
    DevGuard g(c->device);
    PBNG_CUDA(launch_energy_residual(c->prob, c->L, c->work, c->stream), "energy_residual: kernels");
    c->launches += kernels_per_energy_residual();
    std::vector<double> res((size_t)c->nb * 2);
    int32_t flag = 0;
    PBNG_CUDA(cudaMemcpyAsync(res.data(), c->L.results, res.size() * 8, cudaMemcpyDeviceToHost, c->stream),
              "energy_residual: copy");
    PBNG_CUDA(cudaMemcpyAsync(&flag, c->L.flag, 4, cudaMemcpyDeviceToHost, c->stream), "energy_residual: flag");
    PBNG_CUDA(cudaStreamSynchronize(c->stream), "energy_residual: synchronize");
    if (c->comm) {
        // decomposed with the library's transport: global energy = sum over ranks, residual = root of the
        // summed squares (each rank holds its owned tets / constraints / free vertices), fp64 all-reduce
        for (int64_t b = 0; b < c->nb; ++b) res[2 * b + 1] *= res[2 * b + 1];
        double *d = reinterpret_cast<double *>(static_cast<char *>(c->ws) + c->r_allred.off);
        PBNG_CUDA(cudaMemcpyAsync(d, res.data(), res.size() * 8, cudaMemcpyHostToDevice, c->stream), "energy_residual: copy");
        ncclResult_t r = nccl().AllReduce(d, d, res.size(), ncclFloat64, ncclSum, c->comm, c->stream);
        if (r != ncclSuccess) return nccl_fail(r, "energy_residual: all-reduce");
        PBNG_CUDA(cudaMemcpyAsync(res.data(), d, res.size() * 8, cudaMemcpyDeviceToHost, c->stream), "energy_residual: copy");
        PBNG_CUDA(cudaStreamSynchronize(c->stream), "energy_residual: synchronize");
        for (int64_t b = 0; b < c->nb; ++b) res[2 * b + 1] = std::sqrt(res[2 * b + 1]);
    }
    for (int64_t b = 0; b < c->nb; ++b) {
        if (energy_out) energy_out[b] = res[2 * b];
        if (residual_out) residual_out[b] = res[2 * b + 1];
    }
    if (flag & 2) return fail(PBNG_E_CUDA, "peer halo: a neighbour rank's signal did not arrive in time");
    if (flag) return fail(PBNG_E_NONFINITE, "a non-finite position was produced");
    return PBNG_OK;
}

pbng_status pbng_query(pbng_ctx *c, pbng_info *info) {
    if (!c || !info) return fail(PBNG_E_INVALID_ARGUMENT, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->n_vertices = c->nv;
    info->n_tets = c->nt;
    info->n_pinned = (int64_t)c->pinned.size();
    info->n_weak_constraints = (int64_t)c->wc.size();
    info->n_batch = c->nb;
    info->dtype = c->dtype;
    info->model = c->model;
    info->iteration = c->l;
    info->kernel_launches = c->launches;
    info->rank = c->rank;
    info->n_ranks = c->n_ranks;
    if (c->colored) {
        info->n_free = c->n_free;
        info->n_pairs = c->n_pairs;
        info->n_pair_slots = c->n_slots;
        info->n_colours = c->ncol;
        info->sweep_bytes = sweep_bytes_model(c);
        info->accel_bytes = accel_bytes_model(c);
        const double per_pair = c->model == MODEL_FCR ? 130.0 + 700.0 : 130.0;
        info->sweep_flops = (double)c->nb * ((double)c->n_pairs * per_pair + (double)c->n_free * 40.0);
        info->n_local_vertices = c->n_local;
        info->n_ghosts = c->n_local_free - c->n_free;
        info->schedule = effective_schedule(c);
    }
    info->graph_replays = (int32_t)c->dd_graph_replays;
    info->records = !c->colored ? 0 : c->rest_rec ? 2 : c->tab_rec ? 3 : 1;
    return PBNG_OK;
}

pbng_status pbng_set_records(pbng_ctx *c, pbng_records records) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (records != PBNG_RECORDS_AUTO && records != PBNG_RECORDS_STORED && records != PBNG_RECORDS_REST &&
        records != PBNG_RECORDS_TABLE)
        return fail(PBNG_E_INVALID_ARGUMENT, "set_records: unknown record layout");
    if (c->colored) return fail(PBNG_E_BAD_ORDER, "set_records: the record layout is built by pbng_color; call it before");
    c->records = (int)records;
    return PBNG_OK;
}

pbng_status pbng_set_schedule(pbng_ctx *c, pbng_schedule schedule) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (schedule != PBNG_SCHEDULE_AUTO && schedule != PBNG_SCHEDULE_COLOUR_LAUNCHES && schedule != PBNG_SCHEDULE_PIPELINED)
        return fail(PBNG_E_INVALID_ARGUMENT, "set_schedule: unknown schedule");
    if (schedule == PBNG_SCHEDULE_PIPELINED) {
        if (!c->colored) return fail(PBNG_E_NOT_COLORED, "set_schedule: call pbng_color first");
        if (!pipeline_available(c))
            return fail(PBNG_E_INVALID_ARGUMENT, "set_schedule: the pipelined schedule needs an undecomposed context with n_batch < 32");
    }
    if (c->cur_accel >= 0) return fail(PBNG_E_BAD_ORDER, "set_schedule: a colour-by-colour iteration is open");
    c->schedule = (int)schedule;
    return PBNG_OK;
}

pbng_status pbng_set_l2_persistence(pbng_ctx *c, int enable) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->bound) return fail(PBNG_E_BAD_ORDER, "set_l2_persistence: bind a workspace first");
    st = apply_l2_persistence(c, enable);
    if (st == PBNG_OK) c->l2_persist = enable != 0;
    return st;
}

pbng_status pbng_profile_enable(pbng_ctx *c, int enable) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (enable < 0 || enable > 2) return fail(PBNG_E_INVALID_ARGUMENT, "profile_enable: mode must be 0, 1 or 2");
    c->profiling = enable;
    return PBNG_OK;
}

pbng_status pbng_profile_read(pbng_ctx *c, double *sweep_ms, int64_t *sweep_launches) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    DevGuard g(c->device);
    PBNG_CUDA(cudaStreamSynchronize(c->stream), "profile_read: synchronize");
    double total = 0.0;
    int64_t n = 0;
    for (size_t k = 0; k < c->ev_used.size(); ++k) {
        float ms = 0.f;
        PBNG_CUDA(cudaEventElapsedTime(&ms, c->ev_used[k].first, c->ev_used[k].second), "profile_read: elapsed");
        total += ms;
        n += c->ev_launches[k];
        c->ev_free.push_back(c->ev_used[k]);
    }
    if (sweep_ms) *sweep_ms = total;
    if (sweep_launches) *sweep_launches = n;
    c->ev_used.clear();
    c->ev_launches.clear();
    return PBNG_OK;
}

pbng_status pbng_test_polar(pbng_dtype dtype, const double *F, double *R, int64_t n, int device) {
    if (!F || !R || n < 0 || (dtype != PBNG_F32 && dtype != PBNG_F64) || device < 0)
        return fail(PBNG_E_INVALID_ARGUMENT, "test_polar: bad arguments");
    if (n == 0) return PBNG_OK;
    DevGuard g(device);
    double *dF = nullptr, *dR = nullptr;
    const size_t bytes = (size_t)n * 9 * sizeof(double);
    PBNG_CUDA(cudaMalloc(&dF, bytes), "test_polar: cudaMalloc");
    cudaError_t e = cudaMalloc(&dR, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(dF, F, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_polar_test(dtype, dF, dR, n, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(R, dR, bytes, cudaMemcpyDeviceToHost);
    cudaFree(dF);
    if (dR) cudaFree(dR);
    if (e != cudaSuccess) return cuda_fail(e, "test_polar");
    return PBNG_OK;
}

}  // extern "C"

// pbng_update_constraints when the incremental recolouring changed no colour: the
// colour-sorted layout, the pair records and the iterate stay where they are; only the weak-constraint
// arrays (and, for the pipelined schedule, the chunk dependency lists) are rebuilt on the host and written
// into their headroom in the workspace.  Positions, acceleration state and the backward-Euler target are
// kept; new Dirichlet targets are written into the pinned rows (the acceleration state then restarts, as
// with pbng_set_positions).  PBNG_E_OUT_OF_MEMORY = no headroom left (the caller re-lays out).
static pbng_status update_constraints_in_place(pbng_ctx *c, const double *pinned_xyz, const pbng_weak_constraint *wc,
                                               int64_t n_wc) {
    // a free vertex without tets must keep a constraint; the re-layout reports it
    std::vector<char> touched((size_t)c->nv, 0);
    for (int64_t q = 0; q < n_wc; ++q) {
        for (int a = 0; a < wc[q].n0; ++a) touched[wc[q].idx0[a]] = 1;
        for (int a = 0; a < wc[q].n1; ++a) touched[wc[q].idx1[a]] = 1;
    }
    for (int64_t i = 0; i < c->n_free; ++i)
        if (c->h_deg[i] == 0 && !touched[c->int2orig[i]]) return fail(PBNG_E_OUT_OF_MEMORY, "update_constraints: re-layout");
    PhaseTimer T;
    const std::vector<pbng_weak_constraint> old_wc = c->wc;
    const std::vector<int32_t> old_local = c->cons_local;
    const int64_t old_owned = c->n_cons_owned;
    c->wc.assign(wc, wc + n_wc);
    c->cons_local.resize((size_t)n_wc);
    for (int64_t q = 0; q < n_wc; ++q) c->cons_local[q] = (int32_t)q;
    c->n_cons_owned = n_wc;
    if (c->dtype == DT_F64) build_constraint_arrays<double>(c);
    else build_constraint_arrays<float>(c);
    T.lap("in place: constraint arrays");
    const bool deps = pipeline_available(c);
    if (deps) {
        if (c->inc_off.empty()) incidence(c);
        build_pipeline(c, c->inc_off, c->inc);
        T.lap("in place: pipeline dependencies");
    }
    if (c->h_c_n.size() > c->wc_cap || c->h_wc_cid.size() > c->vc_cap || (deps && c->h_deps.size() > c->deps_cap)) {
        c->wc = old_wc;  // no headroom: leave the context as it was for the re-layout
        c->cons_local = old_local;
        c->n_cons_owned = old_owned;
        return fail(PBNG_E_OUT_OF_MEMORY, "update_constraints: re-layout");
    }
    const int64_t np = (int64_t)c->pinned.size();
    if (pinned_xyz) {
        for (int64_t k = 0; k < np; ++k)
            for (int64_t b = 0; b < c->nb; ++b)
                for (int a = 0; a < 3; ++a)
                    c->targets[3 * (b * np + k) + a] = pinned_xyz[3 * (b * np + c->pin_order[k]) + a];
        const size_t s4 = c->real4_size();
        const int64_t npl = (int64_t)c->local_pinned.size();
        for (int64_t b = 0; b < c->nb; ++b)
            for (int64_t k = 0; k < npl; ++k) {
                const double *t = c->targets.data() + 3 * (b * np + c->local_pinned[k]);
                if (c->dtype == DT_F64) put4<double>(c->h_targets, b * npl + k, t[0], t[1], t[2], 0.0);
                else put4<float>(c->h_targets, b * npl + k, t[0], t[1], t[2], 0.0);
            }
        (void)s4;
    }
    Problem &p = c->prob;
    p.has_wc = c->n_vc > 0;
    p.n_cons = c->n_cons_owned;
    const int64_t items = (int64_t)c->tet_local.size() + c->n_cons_owned + c->n_free;
    const int ge_cap = (int)(c->r_part_e.bytes / (8 * (size_t)c->nb));
    p.ge = (int)std::max<int64_t>(1, std::min<int64_t>({(items + kRedBlock - 1) / kRedBlock, 1184, (int64_t)ge_cap}));
    DevGuard g(c->device);
    char *base = static_cast<char *>(c->ws);
    auto up = [&](const Region &r, const void *src, size_t n) -> cudaError_t {
        if (n == 0) return cudaSuccess;
        return cudaMemcpyAsync(base + r.off, src, n, cudaMemcpyHostToDevice, c->stream);
    };
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
    chk(up(c->r_wc_off, c->h_wc_off.data(), c->h_wc_off.size() * 4));
    chk(up(c->r_wc_cid, c->h_wc_cid.data(), c->h_wc_cid.size() * 4));
    chk(up(c->r_wc_d, c->h_wc_d.data(), c->h_wc_d.size()));
    chk(up(c->r_c_n, c->h_c_n.data(), c->h_c_n.size() * 4));
    chk(up(c->r_c_node, c->h_c_node.data(), c->h_c_node.size() * 4));
    chk(up(c->r_c_w, c->h_c_w.data(), c->h_c_w.size()));
    chk(up(c->r_c_anchor, c->h_c_anchor.data(), c->h_c_anchor.size()));
    chk(up(c->r_c_K, c->h_c_K.data(), c->h_c_K.size()));
    if (deps) {
        chk(up(c->r_dep_off, c->h_dep_off.data(), c->h_dep_off.size() * 4));
        chk(up(c->r_deps, c->h_deps.data(), c->h_deps.size() * 4));
    }
    if (pinned_xyz) {
        chk(up(c->r_targets, c->h_targets.data(), c->h_targets.size()));
        if (c->positions_set) {  // pinned rows <- the new targets, free rows kept (through the stage buffer)
            chk(launch_get_positions(c->prob, c->L, c->work, c->stream));
            chk(launch_set_positions(c->prob, c->L, 3, c->stream));
            c->launches += 2;
            c->work = 0;
            c->out = 1;
            c->hist = 2;
            c->l = 0;
            c->hist_valid = true;
        }
    }
    chk(cudaStreamSynchronize(c->stream));  // the host images are rewritten by the next update
    T.lap("in place: upload");
    if (e != cudaSuccess) return cuda_fail(e, "update_constraints: upload");
    c->cur_accel = -1;
    return PBNG_OK;
}

extern "C" {

pbng_status pbng_update_constraints(pbng_ctx *c, const double *pinned_xyz, const pbng_weak_constraint *wc, int64_t n_wc,
                                    int64_t *n_recoloured) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (!c->colored) return fail(PBNG_E_NOT_COLORED, "update_constraints: call pbng_color first");
    if (c->n_ranks > 1) return fail(PBNG_E_INVALID_ARGUMENT, "update_constraints: not supported on a decomposed context");
    if (c->cur_accel >= 0) return fail(PBNG_E_BAD_ORDER, "update_constraints: a colour-by-colour iteration is open");
    if (n_wc < 0 || (n_wc > 0 && !wc)) return fail(PBNG_E_INVALID_ARGUMENT, "update_constraints: bad sizes or pointers");
    const int64_t np = (int64_t)c->pinned.size();
    if (pinned_xyz)
        for (int64_t k = 0; k < (int64_t)c->nb * np * 3; ++k)
            if (!std::isfinite(pinned_xyz[k])) return fail(PBNG_E_INVALID_ARGUMENT, "update_constraints: non-finite target");
    PhaseTimer T;
    pbng_status st = validate_wc(c, wc, n_wc, "update_constraints");
    if (st != PBNG_OK) return st;
    const bool keep = c->bound && c->positions_set;
    int64_t changed = 0;
    try {
        // "newly added" = node set not present among the previous constraints (removed ones only relax)
        std::vector<std::vector<int32_t>> old_nodes, nodes((size_t)n_wc);
        for (const auto &w : c->wc) old_nodes.push_back(distinct_nodes(w));
        std::sort(old_nodes.begin(), old_nodes.end());
        std::vector<char> is_new((size_t)n_wc, 0);
        for (int64_t q = 0; q < n_wc; ++q) {
            nodes[q] = distinct_nodes(wc[q]);
            is_new[q] = !std::binary_search(old_nodes.begin(), old_nodes.end(), nodes[q]);
        }
        T.lap("update: new-constraint sets");
        std::vector<int32_t> col = recolour_incremental(c, nodes, is_new, &changed);
        T.lap("update: incremental recolouring");
        if (changed == 0 && c->bound) {
            st = update_constraints_in_place(c, pinned_xyz, wc, n_wc);
            T.lap("update: in place");
            if (st == PBNG_OK) {
                if (n_recoloured) *n_recoloured = 0;
                return PBNG_OK;
            }
            if (st != PBNG_E_OUT_OF_MEMORY) return st;  // no headroom left: fall through to the re-layout
        }
        // re-layout.  The position, inertial-target and staging regions sit first in the workspace at offsets
        // the re-layout keeps, so the iterate (stage) and the backward-Euler target (stage2) are carried
        // over on the device in original vertex order; nothing goes through the host.
        const double idt2 = c->prob.inv_dt2;
        const bool was_bound = c->bound;
        void *ws = c->ws;
        const uint64_t ws_bytes = c->ws_bytes;
        const size_t fixed_end = c->r_stage2.off + c->r_stage2.bytes;
        if (keep) {
            DevGuard g(c->device);
            Layout L2 = c->L;
            L2.stage = c->stage2;
            if (idt2 > 0.0) PBNG_CUDA(launch_get_positions(c->prob, L2, -1, c->stream), "update_constraints: inertial target");
            PBNG_CUDA(launch_get_positions(c->prob, c->L, c->work, c->stream), "update_constraints: iterate");
            c->launches += idt2 > 0.0 ? 2 : 1;
        }
        c->wc.assign(wc, wc + n_wc);
        if (pinned_xyz)
            for (int64_t k = 0; k < np; ++k)
                for (int64_t b = 0; b < c->nb; ++b)
                    for (int a = 0; a < 3; ++a)
                        c->targets[3 * (b * np + k) + a] = pinned_xyz[3 * (b * np + c->pin_order[k]) + a];
        T.lap("update: save iterate (device)");
        st = colour_and_layout(c, &col);
        T.lap("update: re-layout (host)");
        if (st != PBNG_OK) return st;
        if (n_recoloured) *n_recoloured = changed;
        if (was_bound) {
            if (c->ws_need > ws_bytes) {
                c->prob.inv_dt2 = 0.0;
                return fail(PBNG_E_OUT_OF_MEMORY, "update_constraints: the new layout needs " + std::to_string(c->ws_need) +
                                                      " workspace bytes; bind a larger workspace and set positions");
            }
            if (c->r_stage2.off + c->r_stage2.bytes != fixed_end)
                return fail(PBNG_E_INVALID_ARGUMENT, "update_constraints: position regions moved (internal error)");
            st = bind_layout(c, ws, ws_bytes, !keep);
            if (st != PBNG_OK) return st;
            if (keep) {
                DevGuard g(c->device);
                c->prob.inv_dt2 = idt2;  // carried over: the target is restored from stage2 below
                if (idt2 > 0.0) {
                    Layout L2 = c->L;
                    L2.stage = c->stage2;
                    PBNG_CUDA(launch_set_positions(c->prob, L2, -1, c->stream), "update_constraints: inertial target");
                }
                PBNG_CUDA(launch_set_positions(c->prob, c->L, 3, c->stream), "update_constraints: iterate");
                c->launches += idt2 > 0.0 ? 2 : 1;
                c->work = 0;
                c->out = 1;
                c->hist = 2;
                c->l = 0;
                c->hist_valid = true;
                c->positions_set = true;
                c->cur_accel = -1;
                PBNG_CUDA(cudaStreamSynchronize(c->stream), "update_constraints: synchronize");
                T.lap("update: upload + restore (device)");
            } else {
                c->prob.inv_dt2 = 0.0;
            }
        } else {
            c->prob.inv_dt2 = 0.0;
        }
    } catch (const std::bad_alloc &) {
        return fail(PBNG_E_OUT_OF_MEMORY, "update_constraints: host allocation");
    }
    if (n_recoloured) *n_recoloured = changed;
    return PBNG_OK;
}

pbng_status pbng_get_colours(pbng_ctx *c, int32_t *colour_out, int32_t *n_colours_out) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (!c->colored) return fail(PBNG_E_NOT_COLORED, "get_colours: call pbng_color first");
    if (colour_out) std::memcpy(colour_out, c->colour.data(), (size_t)c->nv * 4);
    if (n_colours_out) *n_colours_out = c->ncol;
    return PBNG_OK;
}

pbng_status pbng_detect_contacts(pbng_ctx *c, int32_t sample, double thickness, double k_n, double k_t,
                                 pbng_weak_constraint *out, int64_t max_out, int64_t *n_out) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (!c->positions_set) return fail(PBNG_E_BAD_ORDER, "detect_contacts: set_positions first");
    if (sample < 0 || sample >= c->nb || !(thickness > 0.0) || !std::isfinite(thickness) || !std::isfinite(k_n) ||
        !std::isfinite(k_t) || k_n < 0.0 || k_t < 0.0 || max_out < 0 || (max_out > 0 && !out) || !n_out)
        return fail(PBNG_E_INVALID_ARGUMENT, "detect_contacts: bad arguments");
    if (c->n_ranks > 1) return fail(PBNG_E_INVALID_ARGUMENT, "detect_contacts: not supported on a decomposed context");
    *n_out = 0;
    if (c->h_sv.empty()) return PBNG_OK;
    DevGuard g(c->device);
    PBNG_CUDA(launch_contacts(c->prob, c->L, c->work, sample, thickness, c->stream), "detect_contacts: kernels");
    c->launches += kernels_per_contacts();
    std::vector<ContactHit> hit(c->h_sv.size());
    PBNG_CUDA(cudaMemcpyAsync(hit.data(), c->L.c_res, hit.size() * sizeof(ContactHit), cudaMemcpyDeviceToHost, c->stream),
              "detect_contacts: copy");
    PBNG_CUDA(cudaStreamSynchronize(c->stream), "detect_contacts: synchronize");
    // one constraint per contacting vertex, in ascending original vertex index
    std::vector<std::pair<int32_t, size_t>> order;
    for (size_t q = 0; q < hit.size(); ++q)
        if (hit[q].tri >= 0) order.push_back({c->int2orig[c->h_sv[q].x], q});
    std::sort(order.begin(), order.end());
    int64_t n = 0;
    for (const auto &o : order) {
        if (n < max_out) {
            const ContactHit &h = hit[o.second];
            pbng_weak_constraint w;
            std::memset(&w, 0, sizeof(w));
            w.n0 = 1;
            w.idx0[0] = o.first;
            w.w0[0] = 1.0;
            w.n1 = 3;
            for (int a = 0; a < 3; ++a) {
                w.idx1[a] = c->surf_orig[3 * (size_t)h.tri + a];
                w.w1[a] = h.bary[a];
            }
            const double *nn = h.normal;  // K = k_n n n^T + k_t (I - n n^T)
            w.K[0] = k_n * nn[0] * nn[0] + k_t * (1.0 - nn[0] * nn[0]);
            w.K[1] = k_n * nn[1] * nn[1] + k_t * (1.0 - nn[1] * nn[1]);
            w.K[2] = k_n * nn[2] * nn[2] + k_t * (1.0 - nn[2] * nn[2]);
            w.K[3] = (k_n - k_t) * nn[0] * nn[1];
            w.K[4] = (k_n - k_t) * nn[1] * nn[2];
            w.K[5] = (k_n - k_t) * nn[0] * nn[2];
            out[n] = w;
        }
        ++n;
    }
    *n_out = n;
    if (n > max_out) return fail(PBNG_E_OUT_OF_MEMORY, "detect_contacts: " + std::to_string(n) + " contacts exceed max_out");
    return PBNG_OK;
}

pbng_status pbng_nccl_unique_id(void *id_out) {
    if (!id_out) return fail(PBNG_E_INVALID_ARGUMENT, "nccl_unique_id: null output");
    const NcclApi &A = nccl();
    if (!A.ok) return fail(PBNG_E_NCCL, "nccl_unique_id: " + A.why);
    ncclUniqueId id;
    ncclResult_t r = A.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "nccl_unique_id");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id_out, &id, sizeof(id));
    return PBNG_OK;
}

pbng_status pbng_partition(pbng_ctx *c, const int32_t *owner, int32_t rank, int32_t n_ranks, const void *nccl_unique_id) {
    if (!c) return fail(PBNG_E_INVALID_ARGUMENT, "null context");
    if (n_ranks > 1) {
        if (!c->on_device()) return fail(PBNG_E_NO_DEVICE, "partition: the NCCL transport needs a device context");
        if (!nccl_unique_id) return fail(PBNG_E_INVALID_ARGUMENT, "partition: null NCCL unique id");
        if (!nccl().ok) return fail(PBNG_E_NCCL, "partition: " + nccl().why);
    }
    pbng_status st = pbng_set_partition(c, owner, rank, n_ranks);
    if (st != PBNG_OK) return st;
    DevGuard g(c->device);
    drop_dd_graph(c);
    peer_release(c);
    if (c->comm) {
        nccl().CommDestroy(c->comm);
        c->comm = nullptr;
    }
    if (n_ranks == 1) return PBNG_OK;
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    ncclResult_t r = nccl().CommInitRank(&comm, n_ranks, id, rank);
    if (r != ncclSuccess) return nccl_fail(r, "partition: ncclCommInitRank");
    c->comm = comm;
    return PBNG_OK;
}

}  // extern "C"

struct pbng_group {
    std::vector<pbng_ctx *> ranks;
    int transport = 0;  // 0: staged device-to-device copies, 1: peer stores
    cudaStream_t side = nullptr, cap = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
};

extern "C" {

pbng_status pbng_group_create(pbng_ctx *const *ctxs, int32_t n_ranks, pbng_group **out) {
    if (!out) return fail(PBNG_E_INVALID_ARGUMENT, "group_create: null output");
    *out = nullptr;
    if (!ctxs || n_ranks < 1 || n_ranks > 64) return fail(PBNG_E_INVALID_ARGUMENT, "group_create: need 1..64 contexts");
    for (int32_t r = 0; r < n_ranks; ++r) {
        pbng_ctx *c = ctxs[r];
        pbng_status st = require_device(c);
        if (st != PBNG_OK) return st;
        if (c->n_ranks != n_ranks || c->rank != r)
            return fail(PBNG_E_INVALID_ARGUMENT, "group_create: ctxs[r] must be rank r of an n_ranks partition");
        if (c->comm) return fail(PBNG_E_INVALID_ARGUMENT, "group_create: context already has an NCCL transport");
        if (!c->colored || !c->bound) return fail(PBNG_E_BAD_ORDER, "group_create: colour and bind every context first");
        const pbng_ctx *c0 = ctxs[0];
        if (c->device != c0->device || c->nb != c0->nb || c->dtype != c0->dtype || c->ncol != c0->ncol)
            return fail(PBNG_E_INVALID_ARGUMENT, "group_create: contexts differ in device, batch, dtype or colouring");
    }
    pbng_group *g = new (std::nothrow) pbng_group();
    if (!g) return fail(PBNG_E_OUT_OF_MEMORY, "group_create: host allocation");
    g->ranks.assign(ctxs, ctxs + n_ranks);
    DevGuard dg(ctxs[0]->device);
    cudaError_t e = cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->cap, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_a, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_b, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        pbng_group_destroy(g);
        return cuda_fail(e, "group_create");
    }
    *out = g;
    return PBNG_OK;
}

pbng_status pbng_group_iterate(pbng_group *g, int32_t n_iterations, pbng_accel accel, double omega, double rho,
                               double gamma) {
    if (!g) return fail(PBNG_E_INVALID_ARGUMENT, "group_iterate: null group");
    if (n_iterations < 0) return fail(PBNG_E_INVALID_ARGUMENT, "group_iterate: negative iteration count");
    pbng_ctx *c0 = g->ranks[0];
    for (pbng_ctx *c : g->ranks) {
        pbng_status st = check_iterate(c, accel, omega, rho, gamma, "group_iterate");
        if (st != PBNG_OK) return st;
        if (c->cur_accel >= 0) return fail(PBNG_E_BAD_ORDER, "group_iterate: a colour-by-colour iteration is open");
        if (c->l != c0->l || c->work != c0->work || c->hist_valid != c0->hist_valid)
            return fail(PBNG_E_BAD_ORDER, "group_iterate: the rank contexts are at different iterations");
    }
    DevGuard dg(c0->device);
    // every rank's launches go to ctxs[0]'s stream for the duration of the call (no kernel waits for another)
    const cudaStream_t main = c0->stream;
    std::vector<cudaStream_t> saved;
    for (pbng_ctx *c : g->ranks) {  // main first waits for the work already queued on every rank's stream
        saved.push_back(c->stream);
        if (c->stream != main) {
            PBNG_CUDA(cudaEventRecord(g->ev_b, c->stream), "group_iterate: event");
            PBNG_CUDA(cudaStreamWaitEvent(main, g->ev_b, 0), "group_iterate: event");
        }
        c->stream = main;
    }
    Exchange X;
    X.ranks = g->ranks;
    X.loopback = true;
    if (g->transport == 1) {
        bool stale = false;
        for (pbng_ctx *c : g->ranks) stale = stale || peer_stale(c);
        if (stale) {
            drop_dd_graph(c0);
            pbng_status ps = peer_setup_group(g->ranks);
            if (ps != PBNG_OK) {
                for (size_t k = 0; k < g->ranks.size(); ++k) g->ranks[k]->stream = saved[k];
                return ps;
            }
        }
        X.peer = true;
    }
    int64_t sweeps = 0;
    pbng_status st = dd_run(c0, X, main, g->side, g->cap, g->ev_a, g->ev_b, n_iterations, accel, omega, rho, gamma,
                            &sweeps, "group_iterate");
    for (size_t k = 0; k < g->ranks.size(); ++k) g->ranks[k]->stream = saved[k];
    if (st == PBNG_OK) {
        cudaEvent_t done = g->ev_a;
        PBNG_CUDA(cudaEventRecord(done, main), "group_iterate: event");
        for (size_t k = 1; k < g->ranks.size(); ++k)
            PBNG_CUDA(cudaStreamWaitEvent(g->ranks[k]->stream, done, 0), "group_iterate: event");
    }
    return st;
}

pbng_status pbng_group_set_transport(pbng_group *g, int32_t transport) {
    if (!g) return fail(PBNG_E_INVALID_ARGUMENT, "group_set_transport: null group");
    if (transport != 0 && transport != 1) return fail(PBNG_E_INVALID_ARGUMENT, "group_set_transport: 0 (copies) or 1 (peer stores)");
    DevGuard dg(g->ranks[0]->device);
    drop_dd_graph(g->ranks[0]);
    if (transport == 0)
        for (pbng_ctx *c : g->ranks) {
            cudaStreamSynchronize(c->stream);
            peer_release(c);
        }
    g->transport = transport;
    return PBNG_OK;
}

pbng_status pbng_enable_peer_halo(pbng_ctx *c, int32_t enable) {
    pbng_status st = require_device(c);
    if (st != PBNG_OK) return st;
    if (c->n_ranks < 2 || !c->comm)
        return fail(PBNG_E_BAD_ORDER, "enable_peer_halo: needs a decomposed context with pbng_partition's communicator");
    if (!c->colored || !c->bound) return fail(PBNG_E_BAD_ORDER, "enable_peer_halo: colour and bind first");
    if (c->n_ranks > kMaxPeers) return fail(PBNG_E_INVALID_ARGUMENT, "enable_peer_halo: at most 64 ranks");
    DevGuard g(c->device);
    PBNG_CUDA(cudaStreamSynchronize(c->stream), "enable_peer_halo: synchronize");
    drop_dd_graph(c);
    if (!enable) {
        peer_release(c);
        return PBNG_OK;
    }
    if (!nccl().AllGather) return fail(PBNG_E_NCCL, "enable_peer_halo: ncclAllGather not available");
    st = peer_setup_comm(c);
    if (st != PBNG_OK) peer_release(c);
    return st;
}

pbng_status pbng_group_destroy(pbng_group *g) {
    if (!g) return PBNG_OK;
    if (!g->ranks.empty()) {
        DevGuard dg(g->ranks[0]->device);
        if (g->side) cudaStreamSynchronize(g->side);
        for (pbng_ctx *c : g->ranks) {
            cudaStreamSynchronize(c->stream);
            peer_release(c);
        }
        drop_dd_graph(g->ranks[0]);
        if (g->side) cudaStreamDestroy(g->side);
        if (g->cap) cudaStreamDestroy(g->cap);
        if (g->ev_a) cudaEventDestroy(g->ev_a);
        if (g->ev_b) cudaEventDestroy(g->ev_b);
    }
    delete g;
    return PBNG_OK;
}

pbng_status pbng_destroy(pbng_ctx *c) {
    if (!c) return PBNG_OK;
    if (c->on_device()) {
        DevGuard g(c->device);
        cudaStreamSynchronize(c->stream);
        clear_l2_persistence(c);  // restore the caller's stream window and the device's persisting limit
        drop_dd_graph(c);
        peer_release(c);
        if (c->comm) nccl().CommDestroy(c->comm);
        if (c->dd_side) cudaStreamDestroy(c->dd_side);
        if (c->dd_cap) cudaStreamDestroy(c->dd_cap);
        if (c->dd_ev_a) cudaEventDestroy(c->dd_ev_a);
        if (c->dd_ev_b) cudaEventDestroy(c->dd_ev_b);
        delete c;
    } else {
        delete c;
    }
    return PBNG_OK;
}

}  // extern "C"
