// pbng_internal.h -- host <-> device launch interface of libpbng (not part of the public C ABI).
//
// The host library (pbng_host.cpp) owns validation, the fp64 rest precompute, the greedy colouring and
// the colour-sorted layout; the kernels (pbng_kernels.cu) own every step of the per-iteration path.
// All pointers below point into the caller-bound workspace.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pbng {

enum { MODEL_NH = 0, MODEL_FCR = 1, MODEL_SNH = 2 };
enum { ACCEL_NONE = 0, ACCEL_SOR = 1, ACCEL_CHEB = 2 };
enum { DT_F32 = 0, DT_F64 = 1 };

constexpr int kChunk = 32;        // vertices per SELL chunk == one warp
#ifndef PBNG_SWEEP_BLOCK
#define PBNG_SWEEP_BLOCK 128
#endif
constexpr int kSweepBlock = PBNG_SWEEP_BLOCK;  // threads per sweep CTA (a multiple of the 32-vertex chunk)
constexpr int kWcMaxNodes = 8;    // distinct nodes per weak constraint
#ifndef PBNG_REC_GROUP
#define PBNG_REC_GROUP 4
#endif
constexpr int kRecGroup = PBNG_REC_GROUP;  // table path records: consecutive slots per lane (4 or 8; group_table_records)
constexpr int kRedBlock = 256;    // threads per reduction CTA

// Pair-record layout (SELL-32, one record per (free vertex i, incident tet e), vertex-major within a
// 32-vertex chunk: slot = chunk_off[chunk] + k * 32 + lane).  For the tet's three OTHER vertices j
// (in slot order) the record holds the internal vertex ids and rest-shape data derived from the
// shape-function gradients g_j (rows of Dm^{-1}); g_i = -(g_1 + g_2 + g_3); VE = V_e E_e.
//   fixed-corotated / stable NH (needs F):
//     f32: rec_id int4 {n1, n2, n3, bits(VE)}; rec_a float4 {g1x g1y g1z g2x}; rec_b float4
//          {g2y g2z g3x g3y}; rec_c float {g3z}                                    -> 52 bytes
//     f64: rec_id int4 {n1, n2, n3, 0}; rec_a double4; rec_b double4; rec_c double2 {g3z, VE} -> 96 bytes
//   Neo-Hookean (needs F g_i, cof(F) g_i, det F only; pbng_kernels.cu Pair<R, MODEL_NH>):
//     f32: rec_id int4 {n1, n2, n3, bits(VE)}; rec_a float4 {s1 s2 s3 detB}, s_j = g_j . g_i -> 32 bytes
//     f64: rec_id int4 {n1, n2, n3, 0}; rec_a double4 {s1 s2 s3 detB}; rec_c double {VE}     -> 56 bytes
// closest boundary triangle of another body found for one free boundary vertex (pbng_detect_contacts)
struct ContactHit {
    int32_t tri = -1, pad = 0;  // boundary-triangle index, -1 = none within the thickness
    double bary[3] = {0, 0, 0};  // closest point = sum bary[a] x_{v_a}
    double normal[3] = {0, 0, 0};  // unit normal of the triangle at the current positions
};

struct Layout {
    int64_t n_vertices = 0, n_slots = 0;  // bounds for the PBNG_DEBUG device asserts
    const int4 *rec_id = nullptr;
    const void *rec_a = nullptr, *rec_b = nullptr, *rec_c = nullptr;
    const int64_t *chunk_off = nullptr;  // [n_chunks + 1]
    const int2 *chunk_v = nullptr;       // [n_chunks] {first internal vertex, vertices in chunk}
    const int32_t *deg = nullptr;        // [n_free] records per vertex
    const int2 *path0 = nullptr;         // [n_free] path mode: slots S1, S2 before the vertex's first record
    const void *rest = nullptr;          // Real4 [n_vertices] rest positions (rest-recompute records) or null
    int path_mode = 0;                   // NH path records: 0 none, 1 stored, 2 rest recompute, 3 table
    int32_t n_tab = 0;                   // table records: distinct rest tuples in rec_a
    const void *fext = nullptr;          // Real4 [n_free] or null (no body force)
    // weak constraints: per free vertex CSR of (constraint id, w0_i - w1_i) in input order
    const int32_t *wc_off = nullptr;     // [n_free + 1]
    const int32_t *wc_cid = nullptr;
    const void *wc_d = nullptr;          // Real
    const int32_t *c_n = nullptr;        // [n_cons] distinct nodes
    const int32_t *c_node = nullptr;     // [n_cons * 8] internal ids
    const void *c_w = nullptr;           // Real [n_cons * 8] combined signed weights w0_j - w1_j
    const void *c_anchor = nullptr;      // Real4 [n_cons] (anchor if side 1 is a fixed point, else 0)
    const void *c_K = nullptr;           // Real [n_cons * 8] xx yy zz xy yz xz (padded)
    // tets for the energy pass: tet_id int4 internal ids; tet_a/b/c Real4 {B00 B01 B02 B10}
    // {B11 B12 B20 B21} {B22 VE V 0}
    const int4 *tet_id = nullptr;
    const void *tet_a = nullptr, *tet_b = nullptr, *tet_c = nullptr;
    const int32_t *int2orig = nullptr;   // [n_vertices]
    const void *targets = nullptr;       // Real4 [n_batch][n_pinned]
    void *xbuf[3] = {nullptr, nullptr, nullptr};  // Real4 [n_batch][x_stride] each
    void *stage = nullptr;               // Real [n_batch][n_vertices][3]
    double *part_e = nullptr;            // [n_batch][ge]
    double *part_r = nullptr;            // [n_batch][gr]
    double *results = nullptr;           // [n_batch][2]
    int32_t *flag = nullptr;             // non-finite flag
    const int32_t *halo_send = nullptr;  // internal ids of the per-(colour, peer) send lists
    const int32_t *halo_recv = nullptr;  // internal ids of the per-(colour, peer) receive lists
    const void *mass = nullptr;          // Real [n_own] lumped masses m_i = sum_e R^0 V_e / 4 (backward Euler)
    void *xtilde = nullptr;              // Real4, position layout: inertial target 2 x^n - x^{n-1}
    // pipelined schedule (sweep_pipe_kernel): per chunk the chunks holding its stencil neighbours, CSR,
    // entry = (chunk << 1) | 1 for an earlier colour (must have finished iteration l), (chunk << 1) for a
    // later colour or the chunk itself (iteration l - 1); done counters [n_batch][n_chunks]; work counter
    // contact detection: boundary triangles {v0, v1, v2, body}, free boundary vertices {vertex, body},
    // hash grid (bucket heads, entries {triangle, next}), per-vertex results, scratch scalars
    const int4 *surf = nullptr;
    const int2 *sv = nullptr;
    int32_t *c_head = nullptr;
    int2 *c_next = nullptr;
    struct ContactHit *c_res = nullptr;
    uint32_t *c_scal = nullptr;
    const int32_t *dep_off = nullptr;    // [n_chunks + 1]
    const int32_t *deps = nullptr;
    int32_t *pipe_flags = nullptr;
    uint64_t *pipe_counter = nullptr;
};

struct Problem {
    int dtype = DT_F32, model = MODEL_NH;
    // n_vertices: vertices held by this context (owned free | ghost free | held pinned); n_global: all
    // vertices of the mesh (the caller's position arrays); n_free: owned + ghost free vertices
    int64_t n_vertices = 0, n_global = 0, n_free = 0, n_pinned = 0, n_tets = 0, n_cons = 0, n_chunks = 0;
    int32_t n_batch = 1;
    int64_t x_stride = 0;  // vertex slots per sample group (positions: pos_index in pbng_kernels.cu)
    int lane_shift = 0;    // 0: [n_batch][x_stride]; 5: [n_batch/32][x_stride][32] (batched, n_batch >= 32)
    double cmu = 0, clam = 0;  // mu_e = cmu * E_e, lambda_e = clam * E_e  (eq:lame)
    double rho_g[3] = {0, 0, 0};  // density * gravity (energy's external-work term)
    bool has_fext = false, has_wc = false;
    int ge = 1, gr = 1;  // energy / residual partial blocks per sample
    int64_t n_own = 0;     // owned free vertices (swept)
    double inv_dt2 = 0;    // backward Euler 1/dt^2 (0: quasistatic)
    int64_t n_surf = 0, n_sv = 0, n_cbuckets = 1;  // contact detection sizes
    int device = 0, sm_count = 0;  // the context's CUDA device and its SM count (queried at bind)
    bool path = false;  // Neo-Hookean pair records in path order (pbng_kernels.cu "path records")
    int path_mode = 0;  // 1 stored rest data, 2 rebuilt from Layout::rest ("rest-recompute"), 3 table of
                        // distinct rest tuples indexed from the record (pbng_kernels.cu load_path_rec)
};

constexpr int kMaxDevices = 64;  // per-device launch caches (pbng_kernels.cu) are indexed by ordinal

struct SweepLaunch {
    int32_t v_begin = 0, n_v = 0;  // colour's internal vertex range
    int64_t chunk_begin = 0;
    int work = 0, out = 1, hist = 2;  // xbuf indices
    int accel = ACCEL_NONE;
    double omega = 1, gamma = 1;  // SOR omega, or Chebyshev omega_{l+1} and gamma
    int split = 1;  // warps sharing one 32-vertex chunk (1, 2, 4 or 8)
    int reverse = 0;  // batched sh-6 launches: walk the sample-group pairs last to first (odd colours)
};

// one launch of the pipelined schedule: n_iter <= kPipeMaxIter whole iterations; iteration l (0-based
// within the launch) reads xbuf[work] (l even) / xbuf[out] (l odd) when accelerated (the buffers swap
// after every accelerated iteration), with blend weight omega[l]
constexpr int kPipeMaxIter = 64;
struct PipeLaunch {
    int n_iter = 0;
    int accel = ACCEL_NONE;
    int work = 0, out = 1, hist = 2;
    int split = 1;  // warps per chunk item (1, 2, 4 or 8), the same as the colour launches use
    double gamma = 1;
    double omega[kPipeMaxIter] = {};
};

// one launch of the windowed persistent schedule of the batched fp32 NH layout (sh 6): n_iter <= kPipeMaxIter
// whole iterations over windows of `window` sample-group pairs; per colour c its vertex range, first chunk
// and block offsets (blocks of kSweepBlock / 32 vertices; blk_off[ncol] = blocks per group pair)
constexpr int kB2MaxColours = 32;
// windowed batched schedule: vertices per warp in one item (an item = kSweepBlock / 32 * kB2WinVpw vertices)
#ifndef PBNG_B2_WIN_VPW
#define PBNG_B2_WIN_VPW 1
#endif
constexpr int kB2WinVpw = PBNG_B2_WIN_VPW;
struct B2Window {
    int n_iter = 0, ncol = 0, window = 4;
    int work = 0, out = 1, hist = 2;
    double gamma = 1;
    double omega[kPipeMaxIter] = {};
    int32_t v_begin[kB2MaxColours] = {}, n_v[kB2MaxColours] = {};
    int64_t chunk_begin[kB2MaxColours] = {};
    int32_t blk_off[kB2MaxColours + 1] = {};
    int32_t prev[kB2MaxColours] = {};  // the previous colour with vertices (cyclic; may be the colour itself)
};

// launchers (pbng_kernels.cu); return cudaGetLastError()
cudaError_t launch_b2_window(const Problem &p, const Layout &L, const B2Window &w, int accel, cudaStream_t st);
// pipelined sweep: the caller zeroes pipe_flags and pipe_counter before each launch
cudaError_t launch_sweep_pipe(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st);
cudaError_t launch_sweep(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st);
cudaError_t launch_set_positions(const Problem &p, const Layout &L, int n_buffers, cudaStream_t st);
cudaError_t launch_get_positions(const Problem &p, const Layout &L, int work, cudaStream_t st);
cudaError_t launch_energy_residual(const Problem &p, const Layout &L, int work, cudaStream_t st);
// halo exchange of one (colour, peer) list: buf is Real4 [n_batch][n][n_fields], fields = work (, out, hist)
cudaError_t launch_halo_pack(const Problem &p, const Layout &L, const int32_t *idx, int64_t n, int n_fields,
                             const int (&bufs)[3], void *buf, cudaStream_t st);
cudaError_t launch_halo_unpack(const Problem &p, const Layout &L, const int32_t *idx, int64_t n, int n_fields,
                               const int (&bufs)[3], const void *buf, cudaStream_t st);
// peer-store halo transport (pbng_kernels.cu "Peer-store halo transport"): one neighbour's rows of one colour,
// stored straight into the neighbour's position buffers
constexpr int kMaxPeers = 64;  // ranks of one decomposition (pbng_group_create's bound)
struct PeerPush {
    const int32_t *idx = nullptr;   // this rank's send rows (internal ids), device
    const int32_t *rows = nullptr;  // the same vertices' ghost rows on the neighbour (its internal ids), device
    int64_t n = 0;
    int nf = 1;                     // fields: work (, out, hist)
    int buf[3] = {0, 1, 2};         // buffer indices of the fields (the ranks rotate their buffers in lockstep)
    int64_t x_stride = 0;
    int sh = 0;
    void *peer_x[3] = {nullptr, nullptr, nullptr};  // the neighbour's xbuf[0..2] through the peer mapping
    int64_t peer_stride = 0;
    int peer_sh = 0;
    int64_t peer_n_vertices = 0;    // vertices the neighbour holds (PBNG_DEBUG bound of `rows`)
    const uint32_t *wait_flag = nullptr;  // own done[q] (null: ordering by the stream alone)
    uint32_t wait_val = 0;
    uint32_t *sig_flag = nullptr;         // the neighbour's pushed[this rank] (null: none)
    uint32_t sig_val = 0;
    uint32_t *counter = nullptr;          // own scratch word, zero between launches
    uint64_t timeout_ns = 0;
};
struct PeerWait {
    const uint32_t *flags = nullptr;
    int n = 0;
    int slot[kMaxPeers] = {};
    uint32_t want = 0;
    uint64_t timeout_ns = 0;
};
struct PeerSignal {
    int n = 0;
    uint32_t *flag[kMaxPeers] = {};
    uint32_t val = 0;
};
cudaError_t launch_halo_push(const Problem &p, const Layout &L, const PeerPush &P, cudaStream_t st);
cudaError_t launch_halo_wait(const Layout &L, const PeerWait &W, cudaStream_t st);
cudaError_t launch_halo_signal(const PeerSignal &S, cudaStream_t st);
cudaError_t launch_halo_sync(const Layout &L, const PeerSignal &S, const PeerWait &W, cudaStream_t st);
int kernels_per_energy_residual();
// contact detection at the positions of buffer `work`, sample `sample`: per free boundary vertex the closest
// boundary triangle of another body within `thickness` (L.c_res); fp64 arithmetic
cudaError_t launch_contacts(const Problem &p, const Layout &L, int work, int sample, double thickness, cudaStream_t st);
int kernels_per_contacts();
cudaError_t launch_polar_test(int dtype, const double *F, double *R, int64_t n, cudaStream_t st);

}  // namespace pbng
