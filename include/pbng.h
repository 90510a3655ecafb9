/*
 * pbng.h -- C ABI of the B200-native Position-Based Nonlinear Gauss-Seidel (PBNG) hot path.
 *
 * Method: Chen, Han, Chen, Teran, "Position-Based Nonlinear Gauss-Seidel for Quasistatic
 * Hyperelasticity", arXiv 2306.09021.  Citations "PAPER.md:N" are lines of the paper text.
 *
 * The calls follow the paper's problem statement: a tetrahedral FEM discretisation,
 * hyperelastic materials, Dirichlet and weak constraints, a node
 * colouring, PBNG iterations with SOR / Chebyshev acceleration
 * (PAPER.md:598-618), and the energy / Newton residual used to judge convergence.
 *
 * Conventions (all functions):
 *  - Every function returns a pbng_status; on failure pbng_last_error() gives a message (thread-local)
 *    and the context is left unchanged (strong guarantee for the setters).  Nothing is thrown across
 *    the ABI.
 *  - Host arrays passed in are copied; the caller keeps ownership.  Device pointers are borrowed for the
 *    duration of the call and used stream-ordered on the context's stream.
 *  - The only device memory the library uses is the workspace the caller allocates and binds
 *    (pbng_bind_workspace); the caller keeps it alive until pbng_destroy.
 *  - Positions are [n_batch][n_vertices][3] in the context dtype (float or double) in the caller's
 *    ORIGINAL vertex order.  Internally the library reorders vertices colour-major.
 *  - Call order: create_mesh -> set_material -> set_constraints -> color -> workspace_bytes ->
 *    bind_workspace -> set_positions -> iterate* / energy_residual / get_positions.  Out-of-order calls
 *    return PBNG_E_BAD_ORDER.  set_material / set_constraints after color invalidate the colouring.
 *  - Functions that return host values (pbng_color, pbng_energy_residual, pbng_synchronize,
 *    pbng_get_positions into host memory) synchronise the stream; all others are asynchronous.
 *  - A context created with device = -1 is host-only: everything up to and including pbng_color and
 *    pbng_query works (CPU tests of the host logic); device calls return PBNG_E_NO_DEVICE.
 */
#ifndef PBNG_H
#define PBNG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbng_ctx pbng_ctx;

typedef enum {
    PBNG_OK = 0,
    PBNG_E_INVALID_ARGUMENT = 1,   /* bad size, null pointer, nu not in [0, 0.5), E <= 0, omega not in (0,2) ... */
    PBNG_E_INDEX_OUT_OF_RANGE = 2, /* a tet / pinned / constraint vertex index outside [0, n_vertices) */
    PBNG_E_DEGENERATE_ELEMENT = 3, /* |det Dm| <= 1e-12 * (mean edge)^3; *bad_index = tet index */
    PBNG_E_ISOLATED_VERTEX = 4,    /* a free vertex with no incident tet and no weak constraint (singular A) */
    PBNG_E_BAD_ORDER = 5,          /* call sequence violated */
    PBNG_E_NOT_COLORED = 6,        /* device call before pbng_color */
    PBNG_E_NONFINITE = 7,          /* a non-finite position was produced (positions left as computed) */
    PBNG_E_CUDA = 8,               /* CUDA runtime error (message in pbng_last_error) */
    PBNG_E_NCCL = 9,               /* NCCL could not be loaded or an NCCL call failed (pbng_partition path) */
    PBNG_E_OUT_OF_MEMORY = 10,     /* host allocation failed or the bound workspace is too small */
    PBNG_E_NO_DEVICE = 11          /* device call on a host-only context */
} pbng_status;

typedef enum { PBNG_F32 = 0, PBNG_F64 = 1 } pbng_dtype;

/* PBNG_NEOHOOKEAN: eq:nh with lambdahat = mu + lambda.
 * PBNG_FIXED_COROTATED: eq:cor, R(F) the closest rotation (polar decomposition).
 * PBNG_STABLE_NEOHOOKEAN: eq:snh read with the cited model's Lame re-parameterisation
 *   mu_s = 4 mu/3, lambda_s = lambda + 5 mu/6 and volume coefficient lambda_s/2 (reading Z18),
 *   which makes it Lame-consistent at F = I as PAPER.md:645 requires.  All models share the modified
 *   Hessian density of eq:mod_hess_dens with the Lame mu, lambda. */
typedef enum { PBNG_NEOHOOKEAN = 0, PBNG_FIXED_COROTATED = 1, PBNG_STABLE_NEOHOOKEAN = 2 } pbng_model;

/* PAPER.md:603-618.  SOR: x^{l+1} = omega (x_PBNG - x^{l-1}) + x^{l-1}.
 * Chebyshev: x^{l+1} = omega_{l+1} (gamma (x_PBNG - x^l) + x^l - x^{l-1}) + x^{l-1},
 * omega_1 = omega_2 = 1, omega_3 = 2/(2 - rho^2), omega_{l+1} = 4/(4 - rho^2 omega_l). */
typedef enum { PBNG_ACCEL_NONE = 0, PBNG_ACCEL_SOR = 1, PBNG_ACCEL_CHEBYSHEV = 2 } pbng_accel;

/* Weak constraint: energy 1/2 C^T K C with C = sum_j w0_j y_{idx0_j} - sum_j w1_j
 * y_{idx1_j}.  n0 in [1,4]; n1 in [0,4], n1 == 0 means side 1 is the fixed point `anchor` (e.g. a
 * rigid-plane contact).  K symmetric PSD given as xx, yy, zz, xy, yz, xz.  176 bytes, no padding. */
typedef struct {
    int32_t n0, n1;
    int32_t idx0[4], idx1[4];
    double w0[4], w1[4];
    double anchor[3];
    double K[6];
} pbng_weak_constraint;

/* Sizes and counters of a coloured context (pbng_query). */
typedef struct {
    int64_t n_vertices, n_tets, n_free, n_pinned, n_weak_constraints;
    int64_t n_pairs;          /* sum over free vertices of incident tets = per-sweep (vertex, tet) records */
    int64_t n_pair_slots;     /* records stored including 32-vertex-chunk padding */
    int32_t n_batch, n_colours;
    int32_t dtype, model;
    int64_t iteration;        /* l: iterations done since the last pbng_set_positions */
    int64_t kernel_launches;  /* kernels this context launched since creation */
    double sweep_bytes;       /* algorithmic HBM bytes of one non-accelerated iteration (all colours, samples) */
    double accel_bytes;       /* extra algorithmic bytes of one SOR / Chebyshev iteration (blend traffic) */
    double sweep_flops;       /* nominal flops of one iteration (per-pair counts) */
    int64_t n_local_vertices; /* vertices held by this context (owned free + ghosts + held pinned) */
    int64_t n_ghosts;         /* free vertices owned by other ranks and held here */
    int32_t rank, n_ranks;
    int32_t schedule;         /* pbng_schedule pbng_iterate uses now (1 colour launches, 2 pipelined) */
    int32_t graph_replays;    /* CUDA-graph replays of decomposed iterate blocks owned by this context */
    int32_t records;          /* pair-record layout built by pbng_color: 1 stored, 2 rest recompute, 3 table */
} pbng_info;

/* How pbng_iterate orders the colour passes (PAPER.md:693-705 fixes only the ORDER: colour after colour,
 * each pass reading the latest values of the other colours).
 * PBNG_SCHEDULE_COLOUR_LAUNCHES: one kernel launch per colour pass (a grid-wide barrier between colours).
 * PBNG_SCHEDULE_PIPELINED: one persistent launch runs up to 64 whole iterations; a 32-vertex chunk starts
 *   as soon as the chunks holding its stencil neighbours have finished the passes it must read after
 *   (earlier colours: this iteration; later colours and itself: the previous one).  Every vertex reads
 *   exactly the values the barrier schedule gives it, so the iterates are bitwise identical; only the
 *   barrier stalls disappear.  Needs an undecomposed context with n_batch < 32.
 * PBNG_SCHEDULE_AUTO (default): pipelined for small problems (few 32-vertex chunks per colour, where the
 *   colour passes are launch / barrier latency bound), colour launches otherwise. */
typedef enum { PBNG_SCHEDULE_AUTO = 0, PBNG_SCHEDULE_COLOUR_LAUNCHES = 1, PBNG_SCHEDULE_PIPELINED = 2 } pbng_schedule;

/* Where the per-(vertex, tet) rest-shape data of the sweep comes from (Dm^{-1} and V^0_e
 * are functions of the rest positions X alone; PAPER.md:570-575 weighs storing per-element data against
 * recomputing it).
 * PBNG_RECORDS_STORED: every record carries its rest data precomputed in fp64 (Neo-Hookean path records:
 *   s'_1..3 = g_j . g_i and det B' in slot order, V_e E_e: 24 B fp32 / 48 B fp64).
 * PBNG_RECORDS_REST: Neo-Hookean path records of an unbatched (n_batch < 32) context carry only the new
 *   neighbour and E_e/6 (8 B fp32 / 16 B fp64); the sweep rebuilds Dm' = [X_a - X_i, X_b - X_i, X_c - X_i]
 *   (slot order) from the rest positions, kept as Real4 in the workspace, and derives g_j, s'_j, det B' and
 *   V_e = |det Dm'|/6 in the compute dtype.  Results agree with STORED within rounding, not bitwise.
 * PBNG_RECORDS_TABLE: the same contexts, when the mesh has at most 256 distinct {s'_1..3, det B'} tuples
 *   (bitwise, in the compute dtype: regular meshes repeat a few element shapes) and fewer than 2^22
 *   vertices: the tuples live in a table in the workspace and each record carries its entry index next to
 *   the neighbour id, plus V_e E_e (8 B fp32 / 16 B fp64).  The sweep reads exactly the values STORED holds,
 *   so the results are bitwise those of STORED.  Falls back to STORED when the table would overflow.
 * REST and TABLE walk path records with one warp per 32-vertex chunk, so requesting them also selects that
 * sweep for problems that would otherwise split a chunk's records over several warps (small problems).
 * Other contexts (fixed-corotated, batched) keep STORED.
 * PBNG_RECORDS_AUTO (default): TABLE where it applies (measured fastest), else STORED. */
typedef enum {
    PBNG_RECORDS_AUTO = 0,
    PBNG_RECORDS_STORED = 1,
    PBNG_RECORDS_REST = 2,
    PBNG_RECORDS_TABLE = 3
} pbng_records;

/* Create a mesh context: rest positions X (n_vertices*3 doubles), tets (n_tets*4
 * int32, any orientation), n_batch >= 1 independent samples sharing mesh, material and colouring
 * (only positions and Dirichlet targets differ), compute dtype, CUDA device ordinal (or -1 for a
 * host-only context) and the cudaStream_t (as an integer; 0 = legacy default stream) used by every
 * later call.  Precomputes Dm^{-1} and V^0_e in fp64.  On PBNG_E_DEGENERATE_ELEMENT or
 * PBNG_E_INDEX_OUT_OF_RANGE *bad_index (optional) receives the offending tet. */
pbng_status pbng_create_mesh(const double *rest_xyz, int64_t n_vertices, const int32_t *tets, int64_t n_tets,
                             int32_t n_batch, pbng_dtype dtype, int device, uintptr_t cuda_stream,
                             pbng_ctx **out, int64_t *bad_index);

/* Material: model, Young's modulus per tet (n_E == n_tets) or uniform (n_E == 1),
 * Poisson ratio nu in [0, 0.5), density R^0 >= 0 and gravity (3 doubles) for the consistent body force
 * f^ext_i = sum_e R^0 g V_e / 4.  Lame parameters by eq:lame. */
pbng_status pbng_set_material(pbng_ctx *ctx, pbng_model model, const double *E, int64_t n_E, double nu,
                              double density, const double gravity[3]);

/* Dirichlet set and weak constraints.  pinned: n_pinned distinct vertex ids;
 * pinned_xyz: targets [n_batch][n_pinned][3] in the order of `pinned`.  wc may be NULL if n_wc == 0. */
pbng_status pbng_set_constraints(pbng_ctx *ctx, const int32_t *pinned, int64_t n_pinned, const double *pinned_xyz,
                                 const pbng_weak_constraint *wc, int64_t n_wc);

/* Greedy node colouring over elements and weak constraints, vertices visited in
 * ascending index, and the colour-sorted device layout it implies.  colour_out (optional, n_vertices
 * int32) receives each vertex's colour, n_colours_out (optional) the number of colours.
 * Fails with PBNG_E_ISOLATED_VERTEX for a free vertex with no incident stencil. */
pbng_status pbng_color(pbng_ctx *ctx, int32_t *colour_out, int32_t *n_colours_out);

/* The same layout from a colouring the caller supplies instead of the greedy one (colours[n_vertices], every
 * vertex, pinned ones included): any node colouring in the sense of PAPER.md:702 -- nodes of one colour share
 * no element and no weak constraint -- gives a valid colour-parallel Gauss-Seidel order,
 * and fewer colours mean fewer, larger colour passes; e.g. (i + j + k) mod 4 on a Kuhn grid,
 * where greedy colouring in index order takes 8.  Validated: PBNG_E_INVALID_ARGUMENT with *bad_index (optional)
 * = the offending vertex, tet, or n_tets + constraint index.  Replaces pbng_color in the call order. */
pbng_status pbng_color_given(pbng_ctx *ctx, const int32_t *colours, int32_t *n_colours_out, int64_t *bad_index);

/* Device bytes the caller must allocate for pbng_bind_workspace (256-byte aligned). */
pbng_status pbng_workspace_bytes(pbng_ctx *ctx, uint64_t *bytes);

/* Bind caller-owned device memory (>= pbng_workspace_bytes, 256-byte aligned) and upload the layout.
 * Synchronises the stream once (set-up only). */
pbng_status pbng_bind_workspace(pbng_ctx *ctx, void *device_ptr, uint64_t bytes);

/* Set x^0 (host or device pointer, [n_batch][n_vertices][3] in the context dtype).  Pinned rows are
 * overwritten by their targets.  Resets the acceleration state: l = 0, x^{-1} = x^0. */
pbng_status pbng_set_positions(pbng_ctx *ctx, const void *x);

/* Backward Euler (eq:fem_be): with dt > 0 every colour pass
 * minimises the incremental potential sum_i m_i/(2 dt^2)|y_i - xtilde_i|^2 + PE(y) - y . f^ext, i.e. adds
 * -m_i (y_i - xtilde_i)/dt^2 to f_i + f^ext_i and m_i/dt^2 I to A, with lumped masses m_ii = int R^0 N_i
 * (needs density > 0) and xtilde = 2 x^n - x^{n-1} ([n_batch][n_vertices][3], context dtype, host or
 * device, original order) supplied by the caller for the step.  The energy / residual of
 * pbng_energy_residual then include the inertia of the (owned) free vertices.  dt = 0 returns to
 * quasistatics.  Asynchronous; requires a bound workspace. */
pbng_status pbng_set_inertia(pbng_ctx *ctx, double dt, const void *xtilde);

/* Current positions x^l into `x_out` (host or device, [n_batch][n_vertices][3], context dtype).
 * Synchronises when x_out is host memory. */
pbng_status pbng_get_positions(pbng_ctx *ctx, void *x_out);

/* n_iterations PBNG iterations: for each colour in order, every free vertex of the
 * colour takes one modified-Newton step x_i += A^{-1}(f_i + f^ext_i) with A of eq:mod_hess; then the
 * acceleration blend.  Continues the acceleration state (l, x^{l-1}) across calls.  omega in (0,2)
 * (SOR), rho in [0,1), gamma in (0,2] (Chebyshev).  Switching from PBNG_ACCEL_NONE to an accelerated
 * mode after l > 0 returns PBNG_E_BAD_ORDER (x^{l-1} was not kept).  Asynchronous. */
pbng_status pbng_iterate(pbng_ctx *ctx, int32_t n_iterations, pbng_accel accel, double omega, double rho,
                         double gamma);

/* Total energy E = sum_e V_e Psi(F_e) + 1/2 sum_c C_c^T K_c C_c - sum_i x_i . f^ext_i (
 * Neo-Hookean shifted so that Psi(I) = 0) and the Newton residual ||(f_i + f^ext_i)_{i free}||_2
 * (PAPER.md:926), per sample, accumulated in fp64 in a fixed order (deterministic).  Either output may
 * be NULL.  Synchronises; returns PBNG_E_NONFINITE if a non-finite position was produced. */
pbng_status pbng_energy_residual(pbng_ctx *ctx, double *energy_out, double *residual_out);

/* ---- fine-grained iteration (domain decomposition drives these; pbng_iterate = loops of them) ---------
 * pbng_sweep_colour: the colour pass `colour` of the current iteration l, with the
 * blend of `accel` fused (the same weights as pbng_iterate).  pbng_end_iteration closes iteration l
 * (x^{l+1} becomes current, l += 1).  Every colour of an iteration must use the same acceleration;
 * mixing returns PBNG_E_BAD_ORDER, as does pbng_iterate while a colour-by-colour iteration is open. */
pbng_status pbng_sweep_colour(pbng_ctx *ctx, int32_t colour, pbng_accel accel, double omega, double rho, double gamma);
pbng_status pbng_end_iteration(pbng_ctx *ctx, pbng_accel accel);
/* pbng_sweep_colour_part: part 1 = the colour's owned vertices that another rank holds as ghosts (laid out
 * first within the colour), part 2 = the others, 0 = both (= pbng_sweep_colour).  Doing part 1, then
 * packing/sending the colour's halo on another stream while part 2 runs, overlaps the exchange with
 * computation (dd.py); the intra-colour order does not change any result.  On an
 * undecomposed context part 1 is empty.
 * pbng_set_stream: the stream later calls of this context use (cudaStream_t as an integer); lets a driver
 * issue the halo pack/unpack on a side stream. */
pbng_status pbng_sweep_colour_part(pbng_ctx *ctx, int32_t colour, int32_t part, pbng_accel accel, double omega,
                                   double rho, double gamma);
pbng_status pbng_set_stream(pbng_ctx *ctx, uintptr_t cuda_stream);

/* ---- domain decomposition -------------------------------------------------------------
 * pbng_set_partition (before pbng_color): owner[v] in [0, n_ranks) for every vertex; this context is rank
 * `rank` (n_ranks <= 64; n_ranks == 1 and owner == NULL is the undecomposed default).  The context then
 * sweeps only its owned free vertices and holds ghost copies of the other vertices its stencils touch;
 * the colouring stays global (identical on every rank), so iterates equal the undecomposed ones bit for
 * bit when the halos are exchanged after every colour pass.  Energy is evaluated for the tets /
 * constraints whose first vertex this rank owns and the residual over owned free vertices, so the
 * global values are the sum over ranks (energy) and the root of the sum of squares (residual).
 * pbng_get_positions writes the rows of held vertices; other rows keep the last pbng_set_positions values.
 *
 * Halo lists: after colour pass k, this rank sends its owned colour-k vertices held by `peer` and receives
 * the colour-k vertices owned by `peer` that it holds; both lists are in ascending original index, so
 * the send list of rank a to b equals the receive list of b from a.  pbng_halo_counts gives the list
 * lengths, pbng_halo_vertices the original vertex ids (host arrays, either may be NULL).
 * pbng_halo_pack gathers the send list into `device_buffer` = Real4 [n_batch][n_send][n_fields], fields =
 * (x_work) or (x_work, x_out, x_hist) for accelerated iterations (n_fields = 3); pbng_halo_unpack
 * scatters a received buffer into the ghost rows.  Both are asynchronous on the context stream; the
 * caller moves the buffers between ranks (bench.py / dd.py: NCCL through torch.distributed). */
pbng_status pbng_set_partition(pbng_ctx *ctx, const int32_t *owner, int32_t rank, int32_t n_ranks);
pbng_status pbng_halo_counts(pbng_ctx *ctx, int32_t colour, int32_t peer, int64_t *n_send, int64_t *n_recv);
pbng_status pbng_halo_vertices(pbng_ctx *ctx, int32_t colour, int32_t peer, int32_t *send_vertices,
                               int32_t *recv_vertices);
pbng_status pbng_halo_pack(pbng_ctx *ctx, int32_t colour, int32_t peer, int32_t n_fields, void *device_buffer);
pbng_status pbng_halo_unpack(pbng_ctx *ctx, int32_t colour, int32_t peer, int32_t n_fields,
                             const void *device_buffer);

/* ---- domain decomposition with the library's own halo transport ----------------
 * The colour loop of PAPER.md:693-705 across ranks: after colour pass k every rank needs the new colour-k
 * values of the ghosts it holds, and nothing else (the colouring is global; PAPER.md:697-698 makes the
 * intra-colour order irrelevant).  With a transport attached, pbng_iterate runs, per colour, entirely
 * inside the library: the colour's halo-send vertices (sweep part 1) on the context stream; then, on a
 * library-owned side stream, pack -> exchange -> unpack while the colour's other vertices (part 2) run on
 * the context stream; the next colour waits for both.  The whole block of n iterations is captured once
 * as a CUDA graph and replayed when pbng_iterate is called again from the same state (same n, blend
 * parameters, iteration index and buffer roles -- e.g. every solve after pbng_set_positions), so the host
 * submits one graph launch per call.  Iterates are bitwise those of the undecomposed context.
 *
 * pbng_nccl_unique_id: writes an NCCL unique id (128 bytes) to id_out (host memory).  Call it on ONE rank
 *   and give the same bytes to every rank (e.g. a torch.distributed broadcast).  PBNG_E_NCCL if NCCL
 *   (libnccl.so.2, loaded at run time; the copy PyTorch already loaded is reused) is not available.
 * pbng_partition (before pbng_color; collective: every rank calls it with the same id): pbng_set_partition
 *   (owner[v] in [0, n_ranks), this context is `rank`) plus an NCCL communicator over the n_ranks ranks on
 *   the context's device, created by the library (ncclCommInitRank).  n_ranks == 1 needs no id (may be
 *   NULL) and creates no communicator.  pbng_energy_residual then returns the GLOBAL energy (sum over
 *   ranks) and residual (root of the summed squares), all-reduced with NCCL in fp64.
 * pbng_group_create / pbng_group_iterate / pbng_group_destroy: the in-process loopback transport (tests
 *   and single-GPU emulation).  ctxs[r] must be rank r of the same n_ranks-rank partition (pbng_set_partition,
 *   no communicator), all on one device, coloured and bound; pbng_group_iterate runs the same per-colour
 *   schedule as the NCCL path for all ranks in turn on ctxs[0]'s stream, the exchange being device-to-device
 *   copies between the ranks' halo buffers.  No kernel ever waits for another rank's kernel.  The group
 *   borrows the contexts (destroy the group first).
 * Halo buffers live in the bound workspace (pbng_workspace_bytes counts them).
 *
 * Peer-store transport (NVLink / NVSwitch peer memory instead of NCCL copies; same iterates bit for bit):
 * pbng_enable_peer_halo(ctx, 1) (collective over pbng_partition's communicator; after pbng_color and
 *   pbng_bind_workspace, again after any re-bind or re-layout -- pbng_iterate returns PBNG_E_BAD_ORDER
 *   otherwise): every rank exports its workspace allocation and a few flag words with cudaIpcGetMemHandle,
 *   the handles and each neighbour's ghost-row lists travel once over NCCL, and the neighbours' memory is
 *   mapped with cudaIpcOpenMemHandle (the workspace must come from cudaMalloc, e.g. PyTorch's default
 *   allocator; the GPUs need peer access).  pbng_iterate then runs, per colour pass E:
 *   part 1 -> per neighbour, on the side stream, ONE kernel { wait until that neighbour has finished pass
 *   E-1 (its `done` flag here); store this rank's boundary rows straight into its ghost rows; raise the
 *   `pushed` flag there } while part 2 runs -> ONE sync kernel { raise the neighbours' `done` flags; wait
 *   until the rows the neighbours store in pass E have landed (their `pushed` flags here) }.
 *   No pack / unpack kernels, no NCCL call per colour (one all-reduce barrier per pbng_iterate call).
 *   A signal that does not arrive within PBNG_PEER_TIMEOUT_MS (environment, default 20000) makes the next
 *   synchronising call return PBNG_E_CUDA instead of hanging.  enable = 0 returns to NCCL send / receive.
 * pbng_group_set_transport(group, 1): the same kernels and flag protocol in the one-GPU loopback group
 *   (the "peer" pointers are the other contexts' buffers; every wait is already satisfied in stream order,
 *   so no kernel spins); 0 = staged copies (default). */
typedef struct pbng_group pbng_group;
pbng_status pbng_nccl_unique_id(void *id_out);
pbng_status pbng_partition(pbng_ctx *ctx, const int32_t *owner_rank, int32_t rank, int32_t n_ranks,
                           const void *nccl_unique_id);
pbng_status pbng_enable_peer_halo(pbng_ctx *ctx, int32_t enable);
pbng_status pbng_group_create(pbng_ctx *const *ctxs, int32_t n_ranks, pbng_group **out);
pbng_status pbng_group_set_transport(pbng_group *group, int32_t transport);
pbng_status pbng_group_iterate(pbng_group *group, int32_t n_iterations, pbng_accel accel, double omega, double rho,
                               double gamma);
pbng_status pbng_group_destroy(pbng_group *group);

/* ---- dynamic weak constraints --------------------------
 * pbng_detect_contacts: proximity detection on the device at the current positions of sample `sample`.
 * Boundary triangles = the tet faces that belong to exactly one tet, in order of (tet index, local face
 * k), face k = the three vertices other than local vertex k in ascending local order, the last two swapped
 * when the rest-state normal (v1 - v0) x (v2 - v0) points towards vertex k; bodies = connected components
 * of tets sharing a vertex.  For every free vertex on a boundary triangle, the boundary triangle of
 * ANOTHER body whose closest point q satisfies |x - q| <= thickness and |x - q|^2 is within
 * 1e-10 thickness^2 of the least such value (closest points on shared edges / vertices tie), the lowest
 * triangle index among those, gives one weak constraint: side 0 = the vertex (weight 1), side 1 = the triangle's
 * vertices with q's barycentric weights, K = k_n n n^T + k_t (I - n n^T), n the triangle's unit normal at
 * the current positions (the paper's collision constraints use k_t = 0).  The paper builds
 * such constraints every time step but gives no detection scheme (reading Z21).  Constraints
 * are written to `out` in ascending vertex index; *n_out = their number (PBNG_E_OUT_OF_MEMORY, with
 * *n_out set, if it exceeds max_out).  fp64 arithmetic; synchronises.  Undecomposed contexts only.
 *
 * pbng_update_constraints: replace the weak constraints (and, if pinned_xyz is not NULL, the Dirichlet
 * targets, [n_batch][n_pinned][3] in the caller's original pinned order) WITHOUT a full recolouring:
 * only the nodes incident to newly added constraints (node sets absent from the previous constraints)
 * are recoloured, in ascending index; each keeps its previous colour unless a node sharing a tet or
 * constraint holds it, else takes the least free colour (reading Z20).
 * The device layout is rebuilt and re-uploaded into the bound workspace and the current iterate is
 * kept (acceleration state reset, as pbng_set_positions; the backward-Euler target is cleared: call
 * pbng_set_inertia again).  If the new layout needs more than the bound workspace, returns
 * PBNG_E_OUT_OF_MEMORY with the context coloured but unbound (bind a workspace of pbng_workspace_bytes
 * and set positions).  *n_recoloured (optional) = nodes whose colour changed.  Synchronises.
 * Works on host-only contexts (recolouring + layout only).  Undecomposed contexts only. */
pbng_status pbng_detect_contacts(pbng_ctx *ctx, int32_t sample, double thickness, double k_n, double k_t,
                                 pbng_weak_constraint *out, int64_t max_out, int64_t *n_out);
pbng_status pbng_update_constraints(pbng_ctx *ctx, const double *pinned_xyz, const pbng_weak_constraint *wc,
                                    int64_t n_wc, int64_t *n_recoloured);
/* The colouring in use (n_vertices int32, optional) and the number of colours (optional): pbng_color's
 * result, or the incremental one after pbng_update_constraints.  Host-only; PBNG_E_NOT_COLORED before
 * pbng_color. */
pbng_status pbng_get_colours(pbng_ctx *ctx, int32_t *colour_out, int32_t *n_colours_out);

/* Wait for the context's stream; PBNG_E_NONFINITE if any iteration produced a non-finite position. */
pbng_status pbng_synchronize(pbng_ctx *ctx);

/* Sizes, byte / flop model and counters. */
pbng_status pbng_query(pbng_ctx *ctx, pbng_info *info);

/* L2 residency of the gathered positions: enable != 0 sets an access-policy window on the context's stream
 * that marks the two position buffers the colour passes gather from (current and next iterate) as
 * persisting in L2 (and sets the device's persisting-L2 limit to their size) when they fit in the device's
 * persisting carve-out (otherwise no window is set: larger buffers would thrash it), so the record
 * stream streaming through L2 does not evict them between colour passes;
 * enable = 0 clears the window.  Affects every kernel later launched on that stream.  Requires a bound
 * workspace; every later pbng_bind_workspace re-applies it. */
pbng_status pbng_set_l2_persistence(pbng_ctx *ctx, int enable);

/* Choose the schedule of pbng_iterate (pbng_schedule above).  PBNG_SCHEDULE_PIPELINED requires a coloured
 * context that supports it (PBNG_E_NOT_COLORED / PBNG_E_INVALID_ARGUMENT otherwise).  Results do not
 * depend on the schedule.  Host-only; may be called between iterations. */
pbng_status pbng_set_schedule(pbng_ctx *ctx, pbng_schedule schedule);

/* Choose the pair-record layout (pbng_records above).  Must precede pbng_color (PBNG_E_BAD_ORDER after it;
 * PBNG_E_INVALID_ARGUMENT for an unknown value).  Host-only. */
pbng_status pbng_set_records(pbng_ctx *ctx, pbng_records records);

/* Timing of the colour-sweep kernel with CUDA events on the context stream (bench.py's roofline).
 * enable = 1: an event pair around every sweep launch; enable = 2: an event pair around the
 * back-to-back sweep launches of each pbng_iterate call (no events between launches, so the kernels
 * are not perturbed; launch gaps are included, a conservative average); 0: off.  pbng_profile_read
 * synchronises, returns the summed time (ms) and the number of sweep launches it covers since the last
 * read, then clears them. */
pbng_status pbng_profile_enable(pbng_ctx *ctx, int enable);
pbng_status pbng_profile_read(pbng_ctx *ctx, double *sweep_ms, int64_t *sweep_launches);

/* TEST HOOK (not on the solve path): the device polar rotation R(F) of eq:cor (closest rotation, det R =
 * +1) for n row-major 3x3 matrices F (host, doubles), computed in `dtype` by the same
 * device routine the fixed-corotated sweep uses; R (host, n*9 doubles).  Allocates its own scratch with
 * cudaMalloc and synchronises (tests only).  Lets the tests pin the routine against numpy's SVD. */
pbng_status pbng_test_polar(pbng_dtype dtype, const double *F, double *R, int64_t n, int device);

/* Release the context (not the workspace, which the caller owns). NULL is a no-op. */
pbng_status pbng_destroy(pbng_ctx *ctx);

/* Message for the last non-OK status returned on this thread (never NULL). */
const char *pbng_last_error(void);

/* ABI version (major * 10000 + minor * 100 + patch). */
int32_t pbng_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PBNG_H */
