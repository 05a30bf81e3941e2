/* crksr.h — C ABI of the B200-native CRK-HACC short-range solver (libcrksr.so).
 *
 * The calls follow the paper's statement of the problem (arxiv 2310.16122): the
 * short-range particle-particle solver that dominates CRK-HACC's GPU time —
 * leaf-pair interaction lists (§5.3 "half-warp" leaves A/B),
 * short-range gravity with a degree-5 grid-force polynomial (PAPER.md:147, 278,
 * 646 HACC_CUDA_POLY_ORDER=5) and the five hot CRK-SPH kernels Geometry,
 * Corrections, Extras, Acceleration, Energy (timers at 503).  The
 * formulas are the readings of SURVEY.md §8(c) O1-O9, listed in DESIGN.md §2.
 *
 * Conventions (every call):
 *  - Pointers inside crk_particles are DEVICE pointers on the ctx's device unless
 *    stated otherwise; the caller owns them.  Arrays are SoA, length n; multi-
 *    component outputs are planes: B[a*n + i], dA[a*n + i], dB[(3a+g)*n + i]
 *    (= d_g B^a), dv[(3a+b)*n + i] (= d_b v^a).
 *  - Calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL =
 *    legacy default stream) except crk_build_lists, which synchronises `stream`
 *    once to size the interaction lists.
 *  - Errors are returned, never thrown: CRK_EINVAL (bad argument or parameter,
 *    nothing launched), CRK_ESTATE (call order violated), CRK_ENOMEM (device
 *    allocation failed), CRK_ECUDA (a CUDA error; crk_last_error has the text).
 *  - A ctx is bound to one device and is not thread-safe; one ctx per stream.
 *  - The ctx owns all scratch (sort buffers, leaves, lists, gas-ordered
 *    intermediates), grown on demand; nothing else is allocated per call.
 */
#ifndef CRKSR_H
#define CRKSR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CRK_OK = 0,
    CRK_EINVAL = -1,
    CRK_ENOMEM = -2,
    CRK_ECUDA = -3,
    CRK_ESTATE = -4,
    CRK_ECAPACITY = -5
} crk_status;

/* Host struct, copied at crk_create. */
typedef struct crk_params {
    double box[3];       /* periodic box per axis, grid units; each a power of two, <= 4096 */
    float rcut2;         /* gravity cutoff^2 (fp32, used verbatim in the O2 predicate) */
    float eps2;          /* Plummer softening added to s = r^2; must be > 0 */
    float poly[6];       /* grid force f_grid(s) = sum_k poly[k] s^k (HACC_CUDA_POLY_ORDER=5) */
    float G;             /* gravity prefactor (cosmology factors folded in) */
    float gamma;         /* adiabatic index of the EOS P = (gamma-1) rho u */
    float av_cl, av_cq;  /* artificial viscosity linear / quadratic coefficients */
    float av_eps2;       /* AV softening eps_AV^2 */
    int32_t leaf_max_i;      /* gravity i-leaf size: 16, 32, 64 or 128 */
    int32_t leaf_max_j;      /* gravity j-leaf size: 8 */
    int32_t leaf_max_gas_i;  /* gas i-leaf size: 16, 32 or 64 */
    int32_t leaf_max_gas_j;  /* gas j-leaf size: 8 */
    double cell_side;    /* chaining-mesh cell side (power of two, <= box/4) */
    int32_t symmetric;   /* kernel-variant bitmask, 0 = every kernel i-centric (each ordered pair
                            evaluated by its i, bit-reproducible); bit 0: gravity evaluates each
                            unordered pair once (Newton's third law) and adds the reactions with
                            float atomics (summation order varies run to run).  Bits 1-2 are
                            ignored (former accel variants).  Same set of terms in every variant. */
    int32_t dom_lo[3], dom_hi[3];  /* owned chaining-mesh cells [dom_lo, dom_hi) per axis (3-D domain
                                      decomposition); all-zero dom_hi = whole box.
                                      With a partial domain, i-leaves (and so every output) exist
                                      only for owned cells; particles in other cells are ghosts
                                      (j-side only: gravity evaluates a pair with a ghost in
                                      the owner's group and drops the reaction). */
    float skin;          /* list skin (grid units, >= 0, < cell_side; whole-box domains only): the
                            leaf-pair lists are built with cutoffs r_c + skin and max H + skin, and
                            after crk_drift steps totalling less than skin/2 per particle
                            crk_refresh renews the position-dependent data without re-sorting or
                            rebuilding the lists.  0 = off. */
    int32_t grav_kernel; /* gravity kernel variant when symmetric & 1 (DESIGN.md §7 and the variant
                            portfolio): 0 = the pipelined warp-independent
                            Newton-3 kernel (the benchmarked default; with 1 and 2 — the same kernel
                            in two other occupancy / staging configurations — the only ones with
                            domain decomposition and count mode, the others fall back to the
                            i-centric kernel there), 6 = warp-independent without the copy
                            pipeline, 7 = CTA-staged,
                            8 = the paper's half-warp XOR-shuffle algorithm.
                            Other values: CRK_EINVAL. */
    int32_t hydro_kernel;/* hydro kernel variant: 0 = default (corrections then extras as two walks of
                            one kernel, accel/du-dt i-centric list walk); 2 = corrections + extras in
                            ONE walk (Extras' sums as moments, 128 registers: slower on c4, 11.4 vs
                            10.5 ms); accel/du-dt variants 4 = 8 lanes per i in 16-warp CTAs,
                            5 = Newton-3 over the lists (whole-box domains), 6 = as 4 with 128-entry
                            staging rounds.  Other: CRK_EINVAL. */
    int32_t nbr_cap;     /* gas neighbour-list capacity per particle (entries; lists built by
                            crk_geometry, walked by corrections, extras and accel): 0 = default
                            (128), < 0 = no lists (every gas pass culls on the fly), else the
                            capacity (rows whose lists overflow it use the on-the-fly kernels). */
} crk_params;

/* Caller-owned particle arrays (device pointers).  Inputs are sorted IN PLACE by
 * crk_build_lists.  Output pointers may be NULL, in which case that output is kept
 * only inside the ctx (the gas-ordered copies used by the next pass). */
typedef struct crk_particles {
    int64_t n;
    float *x, *y, *z;          /* in/out: positions, multiples of q = max(box) 2^-23 in [0, box) */
    float *vx, *vy, *vz;       /* in/out: velocities (kicked by gravity_kick / hydro_accel_dudt) */
    float *m;                  /* in: mass */
    uint8_t *species;          /* in: 0 = dark matter, 1 = gas */
    int64_t *id;               /* in: unique particle ids (tie-break of the sort) */
    float *H, *u;              /* in: gas smoothing length, specific internal energy (u kicked) */
    int32_t *perm;             /* out: perm[k] = input index of the particle now at k */
    float *ax, *ay, *az;       /* out: short-range gravitational acceleration */
    float *V;                  /* out: gas volume (Geometry) */
    float *A, *B, *dA, *dB;    /* out: RK coefficients A, B (3), grad A (3), grad B (9) */
    float *rho, *P, *cs;       /* out: density, pressure, sound speed (Extras) */
    float *dv;                 /* out: velocity gradient (9) (Extras) */
    float *ahx, *ahy, *ahz;    /* out: hydro acceleration (Acceleration) */
    float *dudt;               /* out: du/dt (Energy) */
} crk_particles;

struct crk_ctx;

/* Device views of the lists built by crk_build_lists (valid until the next build
 * or destroy).  Leaf sets: 0 gravity i, 1 gravity j, 2 gas i, 3 gas j.  first[]
 * indexes sorted positions (sets 0,1) or gas ranks (sets 2,3; gas_idx maps a gas
 * rank to its sorted position).  bbox: 6 floats per leaf (lo xyz, hi xyz).
 * Lists: CSR over i-leaves; shift code (sx+1) + 3(sy+1) + 9(sz+1). */
typedef struct crk_lists {
    int64_t n_leaf[4];
    const int32_t* leaf_first[4];
    const int32_t* leaf_count[4];
    const float* leaf_bbox[4];
    const float* leaf_maxh2[4];      /* gas sets only (else NULL) */
    const uint64_t* leaf_cell[4];    /* Morton code of the leaf's cell */
    int64_t n_gas;
    const int32_t* gas_idx;
    int64_t n_entries[2];            /* 0 gravity, 1 hydro */
    const int32_t* row_off[2];
    const int32_t* col[2];
    const int8_t* shift[2];
} crk_lists;

/* Create a solver context on `device`.  Validates params (CRK_EINVAL). */
crk_status crk_create(const crk_params* params, int device, struct crk_ctx** out);
crk_status crk_destroy(struct crk_ctx* ctx);

/* a1 + a2: key -> radix sort -> permute SoA in place -> chaining-
 * mesh cells -> leaves (O3) -> gravity and hydro leaf-pair lists (O4).
 * Fills parts->perm.  Synchronises `stream` once (list sizes). */
crk_status crk_build_lists(struct crk_ctx* ctx, crk_particles* parts, void* stream);

/* a3: a_i = G sum_{j != i, s32 < rcut2} m_j x_ji [(s+eps2)^-3/2 - P5(s)] (O5);
 * writes ax/ay/az and kicks v += dt a (dt = 0: forces only). */
crk_status crk_gravity_kick(struct crk_ctx* ctx, crk_particles* parts, float dt, void* stream);

/* a4 Geometry (upGeo): V_i = 1 / sum_{gas j, s32 < H_i^2, incl. i} W(r_ij, H_i) (O6).
 * Also builds the gas neighbour lists read by the later hydro passes.  Independent of
 * crk_gravity_kick: after crk_build_lists the two may be issued on two different streams
 * (the caller joins them before crk_corrections / crk_corrections_extras, which read the
 * gravity-kicked v); every other call of one ctx must be ordered on one stream. */
crk_status crk_geometry(struct crk_ctx* ctx, crk_particles* parts, void* stream);

/* a5 Corrections (upCor): A, B, grad A, grad B from the moments m0, m1, m2 and their
 * gradients (O7). */
crk_status crk_corrections(struct crk_ctx* ctx, crk_particles* parts, void* stream);

/* a6 Extras (upBarEx): rho = sum m_j W^R_ij, P = (gamma-1) rho u, c = sqrt(gamma P/rho),
 * grad v = sum V_j (v_j - v_i) grad W^R_ij (O8).  Reads the (possibly kicked) v. */
crk_status crk_extras(struct crk_ctx* ctx, crk_particles* parts, void* stream);

/* a5 + a6 in one call, with the results of crk_corrections followed by crk_extras: each
 * gas particle's neighbour list is walked twice by one kernel (Corrections, then Extras
 * with the coefficients just computed, PAPER.md:377 upCor -> upBarEx), sharing the staged
 * neighbour rows (hydro_kernel 2: once, Extras' sums accumulated as moments and combined with
 * the new coefficients in the epilogue).  Call after crk_geometry; leaves the context ready
 * for crk_hydro_accel_dudt.  Reads v and u (as crk_extras does). */
crk_status crk_corrections_extras(struct crk_ctx* ctx, crk_particles* parts, void* stream);

/* Row subset of the following crk_corrections, crk_extras, crk_corrections_extras and
 * crk_hydro_accel_dudt calls (a9, the overlap of the ghost exchange with computation, PAPER.md:252
 * §3.4): 0 = every gas i-leaf row (the default, reset by crk_build_lists),
 * 1 = the rows whose neighbour rows hold no ghost j-leaf (they read no ghost data, so they may run
 * while the R2 / R3 messages are in flight), 2 = the other rows (run after the messages landed).
 * Calls 1 then 2 give the results of one call with 0.  For a whole-box domain every row is
 * interior.  CRK_EINVAL for another value, CRK_ESTATE before crk_build_lists. */
crk_status crk_select_rows(struct crk_ctx* ctx, int32_t which);

/* a7 + a8 Acceleration and Energy (upBarAc, upBarDu): antisymmetrised CRK-SPH momentum
 * and energy derivatives with artificial viscosity (O9); kicks v += dt a_h and
 * u += dt du/dt (dt = 0: derivatives only). */
crk_status crk_hydro_accel_dudt(struct crk_ctx* ctx, crk_particles* parts, float dt, void* stream);

/* ---- sub-cycle steps (readings in DESIGN.md §2 "Sub-cycle") ---- */

/* Time-step limit, written asynchronously to *dt_out (a DEVICE float):
 *   dt = min over particles of  c_acc sqrt(eps / |a_i|)   (eps = sqrt(eps2); a = gravity
 *        acceleration, plus the hydro acceleration for gas)   and, for gas,  c_cfl H_i / c_i
 * (c_i the sound speed of Extras).  A grid-wide float minimum by integer atomicMin on the
 * bits of non-negative floats (the paper's float fetch_min).  Call after
 * crk_hydro_accel_dudt with ax/ay/az, ahx/ahy/ahz, H, species present (sorted order).
 * c_cfl, c_acc > 0 (CRK_EINVAL otherwise).  +inf if every term is infinite. */
crk_status crk_courant_dt(struct crk_ctx* ctx, crk_particles* parts, float c_cfl, float c_acc, float* dt_out,
                          void* stream);

/* Kick: v += dt a (+ a_h for gas), u += dt du/dt (gas), one fp32 fma each, from the
 * caller's ax/ay/az, ahx/ahy/ahz, dudt arrays (all required). */
crk_status crk_kick(struct crk_ctx* ctx, crk_particles* parts, float dt, void* stream);

/* Drift: x' = fl32(x + dt v) rounded to the nearest multiple of q (ties to even) and
 * wrapped into [0, box) — positions stay on the q lattice (O1).  Requires |dt v| < box/2.
 * Invalidates the lists: call crk_build_lists (or, with a skin, crk_refresh) before the next
 * force pass (CRK_ESTATE).  With skin > 0 and lists built, positions are NOT wrapped (they
 * may leave [0, box) by < skin/2; crk_build_lists wraps them) and the drift's largest
 * displacement is added to the displacement bound checked by crk_refresh. */
crk_status crk_drift(struct crk_ctx* ctx, crk_particles* parts, float dt, void* stream);

/* Skin refresh (skin > 0): after crk_drift steps whose displacement bound is < skin/2,
 * renew the position-dependent data (packed positions, leaf boxes, list entry boxes) of
 * the lists built by the last crk_build_lists, keeping the order, leaves and lists: every
 * pair within r_c (or max H) now was within r_c + skin (max H + skin) at the build, so the
 * lists are still supersets and every force pass gives the same results as after a
 * rebuild (same pair terms; the order of summation may differ).  Synchronises `stream`
 * (reads the bound).  CRK_ESTATE if there are no skin lists or the bound is >= skin/2
 * (rebuild).  H must be unchanged since the build. */
crk_status crk_refresh(struct crk_ctx* ctx, crk_particles* parts, void* stream);

/* Smoothing-length update (NEXT-2 H adaptation), after crk_geometry: for every gas
 * particle H_out[i] = factor * sqrt(d2_(k)) (fp32 sqrt and product, correctly rounded),
 * d2_(k) the k_ngb-th smallest O2 squared distance (s32) to another gas particle, selected
 * among its neighbour list.  Exact when d2_(k) < H_i^2 (the list holds every gas particle
 * within H_i); otherwise H_out is an upper bound, or 1.26 H_i (twice the volume) if the list
 * has fewer than k_ngb entries; such particles are counted in n_unconverged (a device int32): rebuild with
 * H = H_out and update again.  H_out: device, length n, sorted order, gas entries written.
 * k_ngb in [1, 127], factor > 0 (CRK_EINVAL); needs the lists (CRK_ESTATE without). */
crk_status crk_update_h(struct crk_ctx* ctx, crk_particles* parts, int32_t k_ngb, float factor, float* H_out,
                        int32_t* n_unconverged, void* stream);

/* Count mode (after SPEC.md:374-382): per-particle integer pair counts,
 * each produced by an integer-payload instantiation of the kernel the corresponding force
 * pass runs (same work items, culls, lists and ownership rules): gravity (j != i,
 * s32 < rcut2) by the configured gravity kernel — the Newton-3 pipelined kernel adds 1 to
 * both particles of every in-range pair it evaluates; gas gather (gas j != i, s32 < H_i^2)
 * counted while walking the neighbour lists the way corrections/extras do; gas symmetric
 * (s32 < max(H_i^2, H_j^2)) while walking them the way accel/du-dt does — with the same
 * on-the-fly fallback for rows whose lists overflowed.  0 for DM.  Outputs are device int32
 * arrays of length n in sorted order.  Needs crk_geometry (it builds the neighbour lists)
 * when the lists are on, else only crk_build_lists. */
crk_status crk_count_pairs(struct crk_ctx* ctx, crk_particles* parts, int32_t* cgrav,
                           int32_t* cgather, int32_t* csym, void* stream);

/* The gas neighbour lists built by crk_geometry (read by corrections, extras and accel/du-dt),
 * decoded: for every gas particle at sorted position i, count[i] = the number of gas particles
 * j (itself included) with s32 < max(H_i^2, H_j^2) — the O2 symmetric predicate, a superset of
 * the gather one — or -1 if its list is incomplete (overflowed the capacity; that particle's row
 * runs the on-the-fly kernels); nbr[i * cap_out + t], t < min(count[i], cap_out), the sorted
 * positions of those neighbours in the list's order.  count = 0 for DM.  count: device int32[n],
 * nbr: device int32[n * cap_out].  CRK_ESTATE before crk_geometry or with the lists off. */
crk_status crk_neighbour_lists(struct crk_ctx* ctx, int32_t cap_out, int32_t* count, int32_t* nbr, void* stream);

/* ---- ghost exchange support ----
 * Cell masks are HOST arrays of ncell[a] bytes per axis; a particle is selected iff its
 * cell (cx, cy, cz) has mask_x[cx] && mask_y[cy] && mask_z[cz].  Selections preserve
 * order.  These calls synchronise `stream` (the count sizes the messages). */

/* Indices (into the given x/y/z arrays, length n) of particles in the masked cells;
 * gas_only != 0 restricts to species == 1.  idx_out: device, capacity n. */
crk_status crk_select_cells(struct crk_ctx* ctx, const float* x, const float* y, const float* z,
                            const uint8_t* species, int gas_only, int64_t n, const uint8_t* mask_x,
                            const uint8_t* mask_y, const uint8_t* mask_z, int32_t* idx_out,
                            int64_t* count_out, void* stream);

/* Gas ranks (ascending) of the gas particles in the masked cells, after crk_build_lists:
 * the same cells give the same particles in the same (key) order on every rank. */
crk_status crk_select_gas(struct crk_ctx* ctx, const uint8_t* mask_x, const uint8_t* mask_y,
                          const uint8_t* mask_z, int32_t* idx_out, int64_t* count_out, void* stream);

/* Device-count variants (no host synchronisation; the weak-scaling exchange of domain.py):
 * the mask is ONE device array of ncell[0] + ncell[1] + ncell[2] bytes (x, then y, then z
 * masks); the number selected is written to *count_dev (device int32). */
crk_status crk_select_cells_dev(struct crk_ctx* ctx, const float* x, const float* y, const float* z,
                                const uint8_t* species, int gas_only, int64_t n, const uint8_t* dmask,
                                int32_t* idx_out, int32_t* count_dev, void* stream);
crk_status crk_select_gas_dev(struct crk_ctx* ctx, const uint8_t* dmask, int32_t* idx_out, int32_t* count_dev,
                              void* stream);
/* crk_select_gas_dev for nsets masks at once (R2/R3 send and receive sets of every peer), after
 * crk_build_lists: set k (mask at dmasks + k * (ncell[0] + ncell[1] + ncell[2])) gets the ascending
 * gas ranks of the gas particles in its cells at idx_out + k * stride (device; entries past stride
 * are dropped: stride >= every set's size keeps them all), its full size at counts_dev[k] (device
 * int32) — the same (key-order) result as nsets calls of crk_select_gas_dev, from one count pass,
 * one scan and one write pass.  1 <= nsets <= 16. */
crk_status crk_select_gas_multi_dev(struct crk_ctx* ctx, const uint8_t* dmasks, int32_t nsets, int32_t* idx_out,
                                    int64_t stride, int32_t* counts_dev, void* stream);

/* R1 selection for every peer in ONE pass over the particles (§3.4: the overload
 * zone each neighbour rank needs): dmasks holds npeers concatenated masks of the layout above
 * (peer q at dmasks + q * (ncell[0] + ncell[1] + ncell[2])); peer q's selected indices go to
 * idx_out + q * stride (device, capacity stride >= n), counts_dev[2 q] = how many were selected,
 * counts_dev[2 q + 1] = how many of those are gas (device int32, zeroed by the call).  Within a
 * peer the order of the indices is NOT deterministic (warp-aggregated atomics); the receiver's
 * build sorts the ghosts by (cell, fine key, id), so nothing downstream depends on it.
 * 1 <= npeers <= 26, else CRK_EINVAL. */
crk_status crk_select_peers_dev(struct crk_ctx* ctx, const float* x, const float* y, const float* z,
                                const uint8_t* species, int64_t n, const uint8_t* dmasks, int32_t npeers,
                                int32_t* idx_out, int64_t stride, int32_t* counts_dev, void* stream);
/* R1 pack of the first min(*count_dev, cap) selected particles (idx: device, capacity cap). */
crk_status crk_pack_particles_dev(struct crk_ctx* ctx, const crk_particles* parts, const int32_t* idx,
                                  const int32_t* count_dev, int64_t cap, void* out, void* stream);

/* The own particles of a sorted local set (after crk_build_lists on own + ghosts, own first
 * in the input): dst rows [0, n_own) = the src rows whose perm (input index) is < n_own, in
 * ascending sorted position, every input field (x y z vx vy vz m H u species id).  The
 * decomposed substep carries its own set this way (§3.4, one rank per GPU over
 * sub-cycles): the next build sorts nearly sorted input and R1 needs no own copy.  src->n =
 * the local set's size, src->perm from the build; dst has room for n_own rows; src and dst
 * must not overlap.  Device pointers; asynchronous on stream. */
crk_status crk_compact_own(struct crk_ctx* ctx, const crk_particles* src, int64_t n_own, crk_particles* dst,
                           void* stream);

/* R1: pack / unpack whole particles as 48-byte records (x y z vx vy vz m H u, species,
 * id).  unpack writes records [0, n) to parts entries [offset, offset + n). */
crk_status crk_pack_particles(struct crk_ctx* ctx, const crk_particles* parts, const int32_t* idx,
                              int64_t n, void* out, void* stream);
crk_status crk_unpack_particles(struct crk_ctx* ctx, crk_particles* parts, int64_t offset, int64_t n,
                                const void* in, void* stream);

/* R2 / R3: pack / unpack per-gas-rank state.  what = 0: volume V (4 bytes; updates the
 * V column of the corrections/extras j-rows), what = 1: the accel record of a7/a8
 * (144 bytes).  Call R2 after crk_geometry, R3 after crk_extras. */
crk_status crk_pack_gas(struct crk_ctx* ctx, int what, const int32_t* idx, int64_t n, void* out,
                        void* stream);
crk_status crk_unpack_gas(struct crk_ctx* ctx, int what, const int32_t* idx, int64_t n, const void* in,
                          void* stream);
/* R2 with velocities (the decomposed substep's R2): per gas rank idx[t], a float4 (V, vx, vy, vz)
 * — the volume and the gravity-kicked velocity its owner's Extras reads (a ghost's R1 copy
 * predates the owner's kick).  unpack writes V into the corrections/extras j-rows and v into
 * the caller's arrays (sorted position gas_idx of the ghost).  After crk_geometry. */
crk_status crk_pack_gas_state(struct crk_ctx* ctx, const crk_particles* parts, const int32_t* idx, int64_t n,
                              void* out, void* stream);
crk_status crk_unpack_gas_state(struct crk_ctx* ctx, crk_particles* parts, const int32_t* idx, int64_t n,
                                const void* in, void* stream);

/* ---- long-range gravity, particle mesh (PAPER.md:146-147 force
 * split; readings in DESIGN.md §2 "Long-range PM") ----
 * Cloud-in-cell deposit on an n_grid^3 periodic mesh, cuFFT real-to-complex transform, the
 * Gaussian-filtered Poisson kernel -4 pi G exp(-k^2 r_s^2) / k^2 (zero mode dropped), a
 * spectral gradient -i k (Nyquist components zeroed), three inverse transforms and
 * cloud-in-cell interpolation: ax/ay/az (device, length n) receive the long-range
 * acceleration of every particle, the counterpart of the short-range force with the same
 * r_s.  Cubic box, n_grid a power of two in [8, 1024], r_s > 0 (CRK_EINVAL otherwise).
 * Independent of crk_ctx; one crk_pm per device; asynchronous on `stream`. */
struct crk_pm;
crk_status crk_pm_create(int n_grid, const double* box, float r_s, float G, int device, struct crk_pm** out);
crk_status crk_pm_destroy(struct crk_pm* pm);
crk_status crk_pm_accel(struct crk_pm* pm, int64_t n, const float* x, const float* y, const float* z,
                        const float* m, float* ax, float* ay, float* az, void* stream);

/* ---- slab-decomposed particle mesh over P ranks ("cuFFT with NCCL
 * all-to-all"; the same operator as crk_pm_accel, DESIGN.md §2 "Distributed PM") ----
 * n = n_grid, nxl = nyl = n / P, nzc = n / 2 + 1; rank r owns the real x-planes
 * [r nxl, (r+1) nxl) and the spectrum's y-rows [r nyl, (r+1) nyl).  The collectives between
 * the calls are the caller's (torch.distributed / NCCL in paper_2310_16122_b200/pm_dist.py):
 *   crk_pm_deposit(mine)             -> rho_full   (n^3 f32, every rank's own particles)
 *   reduce-scatter(sum) rho_full     -> rho_slab   (nxl n n f32: chunk r of the x-major mesh)
 *   crk_pm_slab_forward(rho_slab)    -> send       (P blocks of nxl nyl nzc complex64, block r'
 *                                                   = the y-rows of rank r')
 *   all-to-all(send)                 -> recv       (block r'' = rank r'''s x-planes)
 *   crk_pm_slab_solve(recv)          -> send3      (P blocks of 3 nxl nyl nzc complex64: the
 *                                                   three gradient spectra, x-planes of r'')
 *   all-to-all(send3)                -> recv3
 *   crk_pm_slab_inverse(recv3)       -> acc_slab   (3 nxl n n f32, [c][ixl][iy][iz])
 *   all-gather(acc_slab)             -> acc_full   (P x acc_slab)
 *   crk_pm_interp(acc_full, mine)    -> ax, ay, az (device, length n_mine)
 * All buffers are caller-owned device memory; every call is asynchronous on `stream`.
 * n_grid % nranks != 0, rank out of range or the limits of crk_pm_create -> CRK_EINVAL;
 * crk_pm_accel refuses a slab handle; crk_pm_slab_* and crk_pm_interp refuse a crk_pm_create
 * handle (crk_pm_deposit takes either). */
crk_status crk_pm_slab_create(int n_grid, const double* box, float r_s, float G, int rank, int nranks, int device,
                              struct crk_pm** out);
crk_status crk_pm_deposit(struct crk_pm* pm, int64_t n, const float* x, const float* y, const float* z,
                          const float* m, float* rho_full, void* stream);
crk_status crk_pm_slab_forward(struct crk_pm* pm, const float* rho_slab, void* send, void* stream);
crk_status crk_pm_slab_solve(struct crk_pm* pm, const void* recv, void* send3, void* stream);
crk_status crk_pm_slab_inverse(struct crk_pm* pm, const void* recv3, float* acc_slab, void* stream);
crk_status crk_pm_interp(struct crk_pm* pm, int64_t n, const float* x, const float* y, const float* z,
                         const float* acc_full, float* ax, float* ay, float* az, void* stream);

/* Device views of leaves and lists (after crk_build_lists).  The first call after a build
 * decodes the CSR col / shift arrays from the packed entries (synchronises the device). */
crk_status crk_list_view(struct crk_ctx* ctx, crk_lists* out);

/* Number of kernel launches issued by this ctx since creation (launch accounting). */
int64_t crk_launch_count(struct crk_ctx* ctx);

const char* crk_status_string(crk_status s);
const char* crk_last_error(struct crk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* CRKSR_H */
