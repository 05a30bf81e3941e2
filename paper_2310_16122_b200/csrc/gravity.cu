// gravity.cu — a3: short-range gravity + kick.
//
//   a_i = G sum_{j != i, s32 < rcut2} m_j x_ji [ (s + eps2)^-3/2 - P5(s) ],  v_i += dt a_i
//
// Newtonian minus the fitted grid-force polynomial of order 5 (PAPER.md:147, 278,
// 646 HACC_CUDA_POLY_ORDER=5), Plummer-softened, inside the cutoff.  Per pair: one
// MUFU rsqrt and ~19 FP32 FMA-pipe instructions; FP32-ALU bound.
#include <algorithm>
#include <cstdlib>

#include "pairs.cuh"

namespace crk {

template <bool COUNT>
struct GravPass {
    static constexpr int PAY = 0;
    static constexpr bool SYM = false;
    static constexpr int UNROLL = 4;
    const float4* jrows;  // sorted (x, y, z, m)
    const float4* jpay;
    const float4* xm;
    float rcut2, eps2, G, dt;
    float c0, c1, c2, c3, c4, c5;
    float *ax, *ay, *az, *vx, *vy, *vz;
    int32_t* cnt;

    struct I { float x, y, z; int idx; };
    struct Acc { float ax, ay, az; int n; };

    __device__ void init(Acc& a) const { a.ax = a.ay = a.az = 0.f; a.n = 0; }
    __device__ void load_i(int i, I& s) const {
        const float4 p = xm[i];
        s.x = p.x; s.y = p.y; s.z = p.z; s.idx = i;
    }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I&) const { return rcut2; }
    __device__ float jcut(const float4&) const { return 0.f; }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4*, int j) const {
        const float dx = jp.x - s.x, dy = jp.y - s.y, dz = jp.z - s.z;  // exact (O1)
        const float r2 = s32_of(dx, dy, dz);
        if (COUNT) {
            a.n += (r2 < rcut2 && j != s.idx) ? 1 : 0;
        } else {
            const float ri = rsqrtf(r2 + eps2);
            const float ri3 = ri * ri * ri;
            const float p5 = fmaf(fmaf(fmaf(fmaf(fmaf(c5, r2, c4), r2, c3), r2, c2), r2, c1), r2, c0);
            const float f = r2 < rcut2 ? jp.w * (ri3 - p5) : 0.f;
            a.ax = fmaf(f, dx, a.ax);
            a.ay = fmaf(f, dy, a.ay);
            a.az = fmaf(f, dz, a.az);
        }
    }
    template <int GG>
    __device__ void reduce(Acc& a) const {
        if (COUNT) {
            a.n = slot_sum_i<GG>(a.n);
        } else {
            a.ax = slot_sum<GG>(a.ax);
            a.ay = slot_sum<GG>(a.ay);
            a.az = slot_sum<GG>(a.az);
        }
    }
    __device__ void finish(int i, const I&, const Acc& a) const {
        if (COUNT) {
            cnt[i] = a.n;
            return;
        }
        const float gx = G * a.ax, gy = G * a.ay, gz = G * a.az;
        if (ax) { ax[i] = gx; ay[i] = gy; az[i] = gz; }
        if (dt != 0.f) {
            vx[i] = fmaf(dt, gx, vx[i]);
            vy[i] = fmaf(dt, gy, vy[i]);
            vz[i] = fmaf(dt, gz, vz[i]);
        }
    }
};

// ============================================================== symmetric (Newton-3) variant
// Each unordered pair {i, j} is evaluated once, by the warp of the lower i-group.  Warp
// w of gravity i-leaf a owns the group [gself, gself + ng) with gself = first_a + 16w;
// groups are contiguous ranges of sorted positions, so "j belongs to this or a later
// group" is simply j >= gself.  Lanes own the j-survivors and loop over the warp's 16
// i-particles (shared-memory broadcast); the i-side sums stay in registers for the
// whole row and are reduced once at the end; the j-side reactions (and the final
// i-side sums) go to a float4 accumulator with red.global.add.v4.f32 — the set of
// terms is fixed, their summation order depends on scheduling.  Inside the own group
// the pair is met from both sides, so there only the survivor's (j-side) half counts.
//
// Staging: the whole row (up to ENT entries; longer rows in several rounds) is copied
// into shared memory with 1-D TMA bulk copies (cp.async.bulk, one per j-leaf row of
// packed (x, y, z, m) and one per padded leaf box) completing on one mbarrier; after
// that single wait every warp runs prefilter -> particle filter -> evaluation on its
// own, feeding a 64-entry ring of survivors so that every warp step but the last is full.
namespace symg {
constexpr int RING = 64;
// warps per CTA, row entries per round, row buffers (2 = prefetch), i-particles per warp
template <int NW, int ENT, int NB, int G = 16>
struct Cfg {
struct RowBuf {
    float4 raw[ENT * JMAX];  // TMA: xm rows of the row's j-leaves, JMAX slots per entry
    float4 ebox[ENT][2];     // TMA: padded j-leaf boxes
    float4 eoff[ENT];        // periodic offset (x, y, z) and first (w, as int)
    int ecnt[ENT];
};
struct Smem {
    RowBuf rb[NB];           // NB = 2: the next work item's row streams in during this one
    uint64_t bar[2];
    int next_item;
    float2 inx[NW][G / 2], iny[NW][G / 2], inz[NW][G / 2], im[NW][G / 2];  // (i, i + 8) pairs, -x
    float4 wpos[NW][RING];
    int widx[NW][RING];
    uint16_t went[NW][ENT];
};
};
}  // namespace symg

struct GravSymArgs {
    const float4* xm;
    const uint8_t* gmask;  // per list entry: the i-groups of the row's leaf it can reach (k_entry_masks)
    const float4* box8;  // gravity j-leaf padded boxes
    const int2* erec;    // packed list entries
    const int32_t* row_off;  // row a: entries [row_off[a], row_end[a])
    const int32_t* row_end;
    const int32_t* ifirst;
    const int32_t* icount;
    float4* acc;
    int32_t* cnt;        // count mode: per-particle pair counters (zeroed)
    int* work;           // dynamic work counter (zeroed before the launch)
    int split;           // work items per i-leaf
    int lsplit;          // log2(split) (leaf_max_i / 16 is a power of two: 1, 2, 4 or 8)
    int nitems;
    float L[3];
    float rcut2, eps2;
    float wcut;          // rcut2 * CULL_SLACK (the culls' bound, a kernel parameter so that it stays a constant operand)
    float c0, c1, c2, c3, c4, c5;
    float nc[6];         // -c0 .. -c5 (read straight from the parameter bank in the packed Horner chain)
    // the pipelined kernel's force evaluation in t = s + eps2 (one packed add less per pair, DESIGN.md §2 O5g):
    // -P5(t - eps2) = sum_m ne[m] t^m (coefficients re-expanded in double on the host) and the cutoff
    // t < rce = fl(rcut2 + eps2)
    float ne[6];
    float rce;
    // domain decomposition (grav_pipe_kernel): a particle is owned iff its cell
    // (x / q) >> cs lies in [dlo, dhi) on every axis; ghosts have no i-groups here
    bool partial;
    float inv_q;
    int cs, dlo[3], dhi[3];
};

__device__ __forceinline__ bool grav_owned(const GravSymArgs& A, float x, float y, float z) {
    const int cx = (int)(x * A.inv_q) >> A.cs, cy = (int)(y * A.inv_q) >> A.cs, cz = (int)(z * A.inv_q) >> A.cs;
    return cx >= A.dlo[0] && cx < A.dhi[0] && cy >= A.dlo[1] && cy < A.dhi[1] && cz >= A.dlo[2] && cz < A.dhi[2];
}

// all threads: stage row entries [e0, e0 + nent) of leaf a into buffer rb; every thread
// arrives once on `bar` with the bytes of the copies it issued (barrier count = CTA size)
template <int NW, int ENT, int NB, int GI>
__device__ __forceinline__ void grav_stage(typename symg::Cfg<NW, ENT, NB, GI>::Smem& sm, const GravSymArgs& A, int b, int e0,
                                           int nent) {
    uint32_t bytes = 0;
    for (int t = threadIdx.x; t < nent; t += NW * 32) {
        int first, count, leaf, code;
        unpack_entry(__ldg(A.erec + e0 + t), first, count, leaf, code);
        int sx, sy, sz;
        decode_shift(code, sx, sy, sz);
        sm.rb[b].eoff[t] = make_float4((float)sx * A.L[0], (float)sy * A.L[1], (float)sz * A.L[2], __int_as_float(first));
        sm.rb[b].ecnt[t] = count;
        if (t > 0 && entry_continues(__ldg(A.erec + e0 + t - 1), __ldg(A.erec + e0 + t))) continue;
        const int len = run_length(A.erec, e0 + t, e0 + nent);  // one copy per contiguous run
        int lf, lc, ll, lx;
        unpack_entry(__ldg(A.erec + e0 + t + len - 1), lf, lc, ll, lx);
        const uint32_t pb = (uint32_t)(JMAX * (len - 1) + lc) * 16u;
        bulk_g2s(&sm.rb[b].raw[t * JMAX], A.xm + first, pb, &sm.bar[b]);
        bulk_g2s(&sm.rb[b].ebox[t][0], A.box8 + 2 * (int64_t)leaf, 32u * len, &sm.bar[b]);
        bytes += pb + 32u * len;
    }
    mbar_arrive_expect_tx(&sm.bar[b], bytes);
}

template <int NW, int ENT, int NB, int GI, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) grav_sym_kernel(const GravSymArgs A) {
    using namespace symg;
    constexpr int G = GI;
    static_assert(G == 8 || G == 16, "i-group of 8 or 16");
    using Smem = typename Cfg<NW, ENT, NB, G>::Smem;
    using RowBuf = typename Cfg<NW, ENT, NB, G>::RowBuf;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const float wcut = A.rcut2 * CULL_SLACK;
    const float rc2 = A.rcut2, e2 = A.eps2;
    const float c0 = A.c0, c1 = A.c1, c2 = A.c2, c3 = A.c3, c4 = A.c4, c5 = A.c5;
    float4* wpos = sm.wpos[warp];
    int* widx = sm.widx[warp];
    uint16_t* went = sm.went[warp];

    if (threadIdx.x == 0) {
        mbar_init(&sm.bar[0], NW * 32);
        mbar_init(&sm.bar[1], NW * 32);
        mbar_fence_init();
        sm.next_item = atomicAdd(A.work, 1);
    }
    __syncthreads();
    int w = sm.next_item;
    const int first_w = w;
    uint32_t ph[2] = {0u, 0u};
    int b = 0;
    if (w < A.nitems) {
        const int a0 = w / A.split;
        const int r0 = A.row_off[a0];
        grav_stage<NW, ENT, NB, G>(sm, A, 0, r0, min(ENT, A.row_end[a0] - r0));
    }
    while (w < A.nitems) {
        // claim and prefetch the next work item into the other buffer (free since the
        // barrier that ended the previous item)
        if (threadIdx.x == 0) sm.next_item = atomicAdd(A.work, 1);
        __syncthreads();
        const int wn = sm.next_item;
        if (NB == 2 && wn < A.nitems) {
            const int an = wn / A.split;
            const int rn = A.row_off[an];
            grav_stage<NW, ENT, NB, G>(sm, A, b ^ 1, rn, min(ENT, A.row_end[an] - rn));
        }

        const int a = w / A.split;
        const int ifirst = A.ifirst[a];
        const int icount = A.icount[a];
        const int ibase = (w % A.split * NW + warp) * G;
        const bool wactive = ibase < icount;
        const int gself = ifirst + ibase;  // this warp's group: [gself, gself + ng)
        const int ng = min(G, icount - ibase);
        const int rbeg = A.row_off[a], rend = A.row_end[a];

        float lo[3] = {0.f, 0.f, 0.f}, hi[3] = {0.f, 0.f, 0.f};
        if (wactive) {
            const bool iv = lane < ng;
            float4 p = make_float4(-1e18f, -1e18f, -1e18f, 0.f);  // far sentinel: finite products
            if (iv) p = A.xm[gself + lane];
            if (lane < G) {  // packed (i, i + G/2) pairs of negated positions for FADD2
                const int k = 2 * (lane % (G / 2)) + lane / (G / 2);
                reinterpret_cast<float*>(sm.inx[warp])[k] = -p.x;
                reinterpret_cast<float*>(sm.iny[warp])[k] = -p.y;
                reinterpret_cast<float*>(sm.inz[warp])[k] = -p.z;
                reinterpret_cast<float*>(sm.im[warp])[k] = p.w;
            }
            lo[0] = warp_min(iv ? p.x : INFINITY);
            lo[1] = warp_min(iv ? p.y : INFINITY);
            lo[2] = warp_min(iv ? p.z : INFINITY);
            hi[0] = warp_max(iv ? p.x : -INFINITY);
            hi[1] = warp_max(iv ? p.y : -INFINITY);
            hi[2] = warp_max(iv ? p.z : -INFINITY);
        }
        __syncwarp();
        // i-side sums, packed: component .x is i = k, .y is i = k + G/2
        float2 ax[G / 2], ay[G / 2], az[G / 2];
#pragma unroll
        for (int k = 0; k < G / 2; ++k) ax[k] = ay[k] = az[k] = make_float2(0.f, 0.f);

        // one warp step over ring slots [r0, r0 + n): lane owns one survivor and evaluates
        // its pairs with the group two at a time in packed FP32 (FFMA2 / FADD2 / FMUL2: one
        // issue slot per two pairs; every op still rounds per component, so the O2 predicate
        // is bit-identical to the scalar form)
        auto eval_step = [&](int r0, int n) {
            float4 jp = make_float4(1e18f, 1e18f, 1e18f, 0.f);
            int j = 0;
            if (lane < n) {
                const int s = (r0 + lane) & (RING - 1);
                jp = wpos[s];
                j = widx[s];
            }
            // own group: the i-side half is counted when the partner is the survivor
            const float mj = (j >= gself && j < gself + ng) ? 0.f : jp.w;
            const float2 jx = make_float2(jp.x, jp.x), jy = make_float2(jp.y, jp.y), jz = make_float2(jp.z, jp.z);
            const float2 mj2 = make_float2(mj, mj), e22 = make_float2(e2, e2);
            const float2 n0 = make_float2(-c0, -c0), n1 = make_float2(-c1, -c1), n2 = make_float2(-c2, -c2);
            const float2 n3 = make_float2(-c3, -c3), n4 = make_float2(-c4, -c4), n5 = make_float2(-c5, -c5);
            float2 bx = make_float2(0.f, 0.f), by = bx, bz = bx;
#pragma unroll
            for (int k = 0; k < G / 2; ++k) {
                const float2 dx = __fadd2_rn(jx, sm.inx[warp][k]);  // x_j - x_i, exact (O1)
                const float2 dy = __fadd2_rn(jy, sm.iny[warp][k]);
                const float2 dz = __fadd2_rn(jz, sm.inz[warp][k]);
                const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));  // O2 order
                const float2 re = __fadd2_rn(r2, e22);
                const float2 ri = make_float2(rsqrtf(re.x), rsqrtf(re.y));
                const float2 ri2 = __fmul2_rn(ri, ri);
                float2 np5 = __ffma2_rn(n5, r2, n4);  // -P5(s)
                np5 = __ffma2_rn(np5, r2, n3);
                np5 = __ffma2_rn(np5, r2, n2);
                np5 = __ffma2_rn(np5, r2, n1);
                np5 = __ffma2_rn(np5, r2, n0);
                float2 w = __ffma2_rn(ri2, ri, np5);  // (s + eps2)^-3/2 - P5(s)
                w.x = r2.x < rc2 ? w.x : 0.f;
                w.y = r2.y < rc2 ? w.y : 0.f;
                const float2 wi = __fmul2_rn(mj2, w);  // i-side: a_i += m_j w x_ji
                ax[k] = __ffma2_rn(wi, dx, ax[k]);
                ay[k] = __ffma2_rn(wi, dy, ay[k]);
                az[k] = __ffma2_rn(wi, dz, az[k]);
                const float2 wj = __fmul2_rn(sm.im[warp][k], w);  // j-side: a_j -= m_i w x_ji
                bx = __ffma2_rn(wj, dx, bx);
                by = __ffma2_rn(wj, dy, by);
                bz = __ffma2_rn(wj, dz, bz);
            }
            if (lane < n) red_add_v4(A.acc + j, -(bx.x + bx.y), -(by.x + by.y), -(bz.x + bz.y), 0.f);
        };

        int wr = 0, rd = 0;  // ring write / read counters
        for (int e0 = rbeg; e0 < rend; e0 += ENT) {
            const int nent = min(ENT, rend - e0);
            if (e0 > rbeg || (NB == 1 && e0 == rbeg && w != first_w)) {  // rounds staged in place
                __syncthreads();
                grav_stage<NW, ENT, NB, G>(sm, A, b, e0, nent);
            }
            mbar_wait(&sm.bar[b], ph[b]);
            ph[b] ^= 1u;
            const RowBuf& R = sm.rb[b];
            if (wactive) {
                // (1) leaf prefilter: box-box distance, one lane per entry
                int nsurv = 0;
                for (int e = lane; e - lane < nent; e += 32) {
                    bool ek = false;
                    if (e < nent) {
                        const float4 o = R.eoff[e];
                        const float4 bl = R.ebox[e][0], bh = R.ebox[e][1];
                        const float gx = fmaxf(fmaxf(bl.x + o.x - hi[0], lo[0] - bh.x - o.x), 0.f);
                        const float gy = fmaxf(fmaxf(bl.y + o.y - hi[1], lo[1] - bh.y - o.y), 0.f);
                        const float gz = fmaxf(fmaxf(bl.z + o.z - hi[2], lo[2] - bh.z - o.z), 0.f);
                        // entries wholly below this group own no pair (j < gself)
                        ek = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) < wcut && __float_as_int(o.w) + R.ecnt[e] > gself;
                    }
                    const unsigned em = __ballot_sync(0xffffffffu, ek);
                    if (ek) went[nsurv + __popc(em & ((1u << lane) - 1u))] = (uint16_t)e;
                    nsurv += __popc(em);
                }
                __syncwarp();
                // (2) particle filter, 32/JMAX entries per step, into the survivor ring
                for (int q0 = 0; q0 < nsurv; q0 += 32 / JMAX) {
                    const int qe = q0 + lane / JMAX;
                    const int kk = lane % JMAX;
                    const int e = went[qe < nsurv ? qe : 0];
                    const float4 o = R.eoff[e];
                    float4 p = R.raw[e * JMAX + kk];
                    p.x += o.x; p.y += o.y; p.z += o.z;  // exact (O1)
                    const int j = __float_as_int(o.w) + kk;
                    const bool keep = qe < nsurv && kk < R.ecnt[e] && j >= gself &&
                                      box_dist2(p.x, p.y, p.z, lo, hi) < wcut;
                    const unsigned msk = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        const int s = (wr + __popc(msk & ((1u << lane) - 1u))) & (RING - 1);
                        wpos[s] = p;
                        widx[s] = j;
                    }
                    wr += __popc(msk);
                    __syncwarp();
                    if (wr - rd >= 32) {
                        eval_step(rd, 32);
                        rd += 32;
                        __syncwarp();
                    }
                }
            }
        }
        if (wactive) {
            if (wr > rd) eval_step(rd, wr - rd);
            // transposed (reduce-scatter) sum of the 16 x 3 i-side values over the warp:
            // after the halving steps over lane bits 4..1, lane l holds i = l >> 1 (48 shuffles
            // instead of 48 full warp sums)
            float v[3][G];
#pragma unroll
            for (int k = 0; k < G / 2; ++k) {
                v[0][k] = ax[k].x; v[0][k + G / 2] = ax[k].y;
                v[1][k] = ay[k].x; v[1][k + G / 2] = ay[k].y;
                v[2][k] = az[k].x; v[2][k + G / 2] = az[k].y;
            }
#pragma unroll
            for (int h = G / 2; h >= 1; h >>= 1) {  // lane bit 2h <-> i bit h (G = 16: lane bits 16, 8, 4, 2)
                const bool up = lane & (2 * h);
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int k = 0; k < h; ++k) {
                        const float send = up ? v[c][k] : v[c][k + h];
                        const float keep = up ? v[c][k + h] : v[c][k];
                        v[c][k] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
                    }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                v[c][0] += __shfl_xor_sync(0xffffffffu, v[c][0], 1);
#pragma unroll
                for (int o = 4 * G; o < 32; o <<= 1) v[c][0] += __shfl_xor_sync(0xffffffffu, v[c][0], o);
            }
            const int iq = (lane >> 1) & (G - 1);
            if ((lane & 1) == 0 && lane < 2 * G && iq < ng) red_add_v4(A.acc + gself + iq, v[0][0], v[1][0], v[2][0], 0.f);
        }
        __syncthreads();  // buffer b is free for the item after next
        if (NB == 2) b ^= 1;
        w = wn;
    }
}

// ------------------------------------------------------------ warp-independent variant
// Same pair arithmetic and Newton-3 ownership as grav_sym_kernel, but every warp runs its
// own work items (one 16-particle i-group of a gravity i-leaf) with no CTA barrier and no
// shared row staging: lanes read their row's list entries and j-leaf boxes straight from
// L2 (one entry per lane), cull them against the group's box, load the surviving leaves'
// particles with coalesced 128-byte reads (8 lanes per leaf) and cull them again, and the
// survivors feed the per-warp ring and packed evaluation.  Work items are claimed one warp
// at a time from a global counter, so a slow group never holds up a CTA.
namespace symw {
constexpr int G = 16, RING = 128, NW = 4;
struct WarpSm {
    float4 wpos[RING];
    int widx[RING];
    float2 inx[G / 2], iny[G / 2], inz[G / 2], im[G / 2];  // (i, i + 8) pairs, -x
    float4 woff[32];                                        // surviving entries: shift, first (w)
    int wcnt[32];
};
}  // namespace symw

__global__ void __launch_bounds__(symw::NW * 32, 16 / symw::NW) grav_warp_kernel(const GravSymArgs A) {
    using namespace symw;
    __shared__ WarpSm wsm[NW];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    WarpSm& S = wsm[warp];
    const float wcut = A.rcut2 * CULL_SLACK;
    const float rc2 = A.rcut2, e2 = A.eps2;
    const float c0 = A.c0, c1 = A.c1, c2 = A.c2, c3 = A.c3, c4 = A.c4, c5 = A.c5;
    const unsigned below = (1u << lane) - 1u;

    while (true) {
        int w = 0;
        if (lane == 0) w = atomicAdd(A.work, 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= A.nitems) break;
        const int a = w / A.split;
        const int icount = __ldg(A.icount + a);
        const int ibase = (w % A.split) * G;
        if (ibase >= icount) continue;
        const int gself = __ldg(A.ifirst + a) + ibase;  // this warp's group: [gself, gself + ng)
        const int ng = min(G, icount - ibase);
        const int rbeg = __ldg(A.row_off + a), rend = __ldg(A.row_end + a);

        float lo[3], hi[3];  // the group's box (nlh: (-lo, -hi) per axis, packed for the particle cull)
        {
            const bool iv = lane < ng;
            float4 p = make_float4(-1e18f, -1e18f, -1e18f, 0.f);  // far sentinel: finite products
            if (iv) p = __ldg(A.xm + gself + lane);
            if (lane < G) {  // packed (i, i + G/2) pairs of negated positions for FADD2
                const int k = 2 * (lane % (G / 2)) + lane / (G / 2);
                reinterpret_cast<float*>(S.inx)[k] = -p.x;
                reinterpret_cast<float*>(S.iny)[k] = -p.y;
                reinterpret_cast<float*>(S.inz)[k] = -p.z;
                reinterpret_cast<float*>(S.im)[k] = p.w;
            }
            lo[0] = warp_min(iv ? p.x : INFINITY);
            lo[1] = warp_min(iv ? p.y : INFINITY);
            lo[2] = warp_min(iv ? p.z : INFINITY);
            hi[0] = warp_max(iv ? p.x : -INFINITY);
            hi[1] = warp_max(iv ? p.y : -INFINITY);
            hi[2] = warp_max(iv ? p.z : -INFINITY);
        }
        __syncwarp();
        float2 ax[G / 2], ay[G / 2], az[G / 2];
#pragma unroll
        for (int k = 0; k < G / 2; ++k) ax[k] = ay[k] = az[k] = make_float2(0.f, 0.f);

        auto eval_step = [&](int r0, int n) {
            float4 jp = make_float4(1e18f, 1e18f, 1e18f, 0.f);
            int j = 0;
            if (lane < n) {
                const int s = (r0 + lane) & (RING - 1);
                jp = S.wpos[s];
                j = S.widx[s];
            }
            // own group: the i-side half is counted when the partner is the survivor
            const float mj = (j >= gself && j < gself + ng) ? 0.f : jp.w;
            const float2 jx = make_float2(jp.x, jp.x), jy = make_float2(jp.y, jp.y), jz = make_float2(jp.z, jp.z);
            const float2 mj2 = make_float2(mj, mj), e22 = make_float2(e2, e2);
            const float2 n0 = make_float2(-c0, -c0), n1 = make_float2(-c1, -c1), n2 = make_float2(-c2, -c2);
            const float2 n3 = make_float2(-c3, -c3), n4 = make_float2(-c4, -c4), n5 = make_float2(-c5, -c5);
            float2 bx = make_float2(0.f, 0.f), by = bx, bz = bx;
#pragma unroll
            for (int k = 0; k < G / 2; ++k) {
                const float2 dx = __fadd2_rn(jx, S.inx[k]);  // x_j - x_i, exact (O1)
                const float2 dy = __fadd2_rn(jy, S.iny[k]);
                const float2 dz = __fadd2_rn(jz, S.inz[k]);
                const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));  // O2 order
                const float2 re = __fadd2_rn(r2, e22);
                const float2 ri = make_float2(rsqrtf(re.x), rsqrtf(re.y));
                const float2 ri2 = __fmul2_rn(ri, ri);
                float2 np5 = __ffma2_rn(n5, r2, n4);  // -P5(s)
                np5 = __ffma2_rn(np5, r2, n3);
                np5 = __ffma2_rn(np5, r2, n2);
                np5 = __ffma2_rn(np5, r2, n1);
                np5 = __ffma2_rn(np5, r2, n0);
                float2 wv = __ffma2_rn(ri2, ri, np5);  // (s + eps2)^-3/2 - P5(s)
                wv.x = r2.x < rc2 ? wv.x : 0.f;
                wv.y = r2.y < rc2 ? wv.y : 0.f;
                const float2 wi = __fmul2_rn(mj2, wv);  // i-side: a_i += m_j w x_ji
                ax[k] = __ffma2_rn(wi, dx, ax[k]);
                ay[k] = __ffma2_rn(wi, dy, ay[k]);
                az[k] = __ffma2_rn(wi, dz, az[k]);
                const float2 wj = __fmul2_rn(S.im[k], wv);  // j-side: a_j -= m_i w x_ji
                bx = __ffma2_rn(wj, dx, bx);
                by = __ffma2_rn(wj, dy, by);
                bz = __ffma2_rn(wj, dz, bz);
            }
            if (lane < n) red_add_v4(A.acc + j, -(bx.x + bx.y), -(by.x + by.y), -(bz.x + bz.y), 0.f);
        };

        int wr = 0, rd = 0;
        for (int e0 = rbeg; e0 < rend; e0 += 32) {
            // (1) entry cull: one list entry per lane, box-box distance to the group's box
            const int e = e0 + lane;
            bool ek = false;
            float4 off = make_float4(0.f, 0.f, 0.f, 0.f);
            int cnt = 0;
            if (e < rend) {
                int first, leaf, code;
                unpack_entry(__ldg(A.erec + e), first, cnt, leaf, code);
                int sx, sy, sz;
                decode_shift(code, sx, sy, sz);
                off = make_float4((float)sx * A.L[0], (float)sy * A.L[1], (float)sz * A.L[2], __int_as_float(first));
                if (first + cnt > gself) {  // entries wholly below this group own no pair (j < gself)
                    const float4 bl = __ldg(A.box8 + 2 * (int64_t)leaf), bh = __ldg(A.box8 + 2 * (int64_t)leaf + 1);
                    const float gx = fmaxf(fmaxf(bl.x + off.x - hi[0], lo[0] - bh.x - off.x), 0.f);
                    const float gy = fmaxf(fmaxf(bl.y + off.y - hi[1], lo[1] - bh.y - off.y), 0.f);
                    const float gz = fmaxf(fmaxf(bl.z + off.z - hi[2], lo[2] - bh.z - off.z), 0.f);
                    ek = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) < wcut;
                }
            }
            const unsigned em = __ballot_sync(0xffffffffu, ek);
            if (ek) {
                const int q = __popc(em & below);
                S.woff[q] = off;
                S.wcnt[q] = cnt;
            }
            const int nsurv = __popc(em);
            __syncwarp();
            // (2) particle cull, 4 leaves per load step, two steps' loads in flight
            for (int q0 = 0; q0 < nsurv; q0 += 8) {
                float4 pp[2];
                int jj[2];
                bool vv[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int qe = q0 + 4 * u + lane / JMAX;
                    const int kk = lane % JMAX;
                    const int qc = qe < nsurv ? qe : 0;
                    const float4 o = S.woff[qc];
                    jj[u] = __float_as_int(o.w) + kk;
                    vv[u] = qe < nsurv && kk < S.wcnt[qc] && jj[u] >= gself;
                    pp[u] = vv[u] ? __ldg(A.xm + jj[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
                    pp[u].x += o.x; pp[u].y += o.y; pp[u].z += o.z;  // exact (O1)
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const bool keep = vv[u] && box_dist2(pp[u].x, pp[u].y, pp[u].z, lo, hi) < wcut;
                    const unsigned msk = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        const int s = (wr + __popc(msk & below)) & (RING - 1);
                        S.wpos[s] = pp[u];
                        S.widx[s] = jj[u];
                    }
                    wr += __popc(msk);
                }
                __syncwarp();
                while (wr - rd >= 32) {
                    eval_step(rd, 32);
                    rd += 32;
                }
                __syncwarp();
            }
        }
        if (wr > rd) eval_step(rd, wr - rd);
        // transposed (reduce-scatter) sum of the 16 x 3 i-side values; lane l ends with i = l >> 1
        float v[3][G];
#pragma unroll
        for (int k = 0; k < G / 2; ++k) {
            v[0][k] = ax[k].x; v[0][k + G / 2] = ax[k].y;
            v[1][k] = ay[k].x; v[1][k + G / 2] = ay[k].y;
            v[2][k] = az[k].x; v[2][k + G / 2] = az[k].y;
        }
#pragma unroll
        for (int h = G / 2; h >= 1; h >>= 1) {
            const bool up = lane & (2 * h);
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int k = 0; k < h; ++k) {
                    const float send = up ? v[c][k] : v[c][k + h];
                    const float keep = up ? v[c][k + h] : v[c][k];
                    v[c][k] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
                }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c][0] += __shfl_xor_sync(0xffffffffu, v[c][0], 1);
        if ((lane & 1) == 0 && (lane >> 1) < ng) red_add_v4(A.acc + gself + (lane >> 1), v[0][0], v[1][0], v[2][0], 0.f);
        __syncwarp();  // the group's shared i-data is rewritten by the next item
    }
}

// ------------------------------------------------------------ half-warp shuffle variant
// The paper's "half-warp" algorithm (Figs. half-warp-layout and
// half-warp-shuffle), kept as a measured variant (
// crk_params.grav_kernel = 8): lanes 0-15 hold the 16 i-particles of a work item, lanes 16-31 the
// particles of two surviving j-leaves (8 lanes each).  In step k = 0..15 every lane
// exchanges its particle with lane ^ (16 | k) by __shfl_xor_sync and adds the force its
// partner exerts on its own particle: lane l < 16 evaluates (i_l, j), its partner the
// reverse (j, i_l), so each pair is evaluated twice (once per direction, no per-pair atomics)
// and the j-side sums reach memory once per j-leaf pair with red.global.add.  A pair
// (p, q) belongs to the item of its lower index (the other item skips it), the same
// Newton-3 ownership as the other symmetric kernels.  No domain decomposition.
namespace symh {
constexpr int G = 16, NW = 4;
struct WarpSm {
    float4 woff[32];  // surviving entries: shift, first (w)
    int wcnt[32];
};
}  // namespace symh

__global__ void __launch_bounds__(symh::NW * 32, 16 / symh::NW) grav_halfwarp_kernel(const GravSymArgs A) {
    using namespace symh;
    __shared__ WarpSm wsm[NW];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    WarpSm& S = wsm[warp];
    const float wcut = A.rcut2 * CULL_SLACK;
    const float rc2 = A.rcut2, e2 = A.eps2;
    const float c0 = A.c0, c1 = A.c1, c2 = A.c2, c3 = A.c3, c4 = A.c4, c5 = A.c5;
    const unsigned below = (1u << lane) - 1u;
    const bool lower = lane < 16;

    while (true) {
        int w = 0;
        if (lane == 0) w = atomicAdd(A.work, 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= A.nitems) break;
        const int a = w / A.split;
        const int icount = __ldg(A.icount + a);
        const int ibase = (w % A.split) * G;
        if (ibase >= icount) continue;
        const int gself = __ldg(A.ifirst + a) + ibase;
        const int ng = min(G, icount - ibase);
        const int rbeg = __ldg(A.row_off + a), rend = __ldg(A.row_end + a);

        // lower half: the item's i-particles (index -1: no particle)
        float4 ip = make_float4(0.f, 0.f, 0.f, 0.f);
        int iidx = -1;
        if (lower && lane < ng) {
            iidx = gself + lane;
            ip = __ldg(A.xm + iidx);
        }
        float lo[3], hi[3];  // the group's box (nlh: (-lo, -hi) per axis, packed for the particle cull)
        {
            const bool iv = iidx >= 0;
            lo[0] = warp_min(iv ? ip.x : INFINITY);
            lo[1] = warp_min(iv ? ip.y : INFINITY);
            lo[2] = warp_min(iv ? ip.z : INFINITY);
            hi[0] = warp_max(iv ? ip.x : -INFINITY);
            hi[1] = warp_max(iv ? ip.y : -INFINITY);
            hi[2] = warp_max(iv ? ip.z : -INFINITY);
        }
        float acc[3] = {0.f, 0.f, 0.f};  // lower: the i-particle (whole item); upper: per instance

        for (int e0 = rbeg; e0 < rend; e0 += 32) {
            // entry cull (as grav_warp_kernel): one list entry per lane against the item's box
            const int e = e0 + lane;
            bool ek = false;
            float4 off = make_float4(0.f, 0.f, 0.f, 0.f);
            int cnt = 0;
            if (e < rend) {
                int first, leaf, code;
                unpack_entry(__ldg(A.erec + e), first, cnt, leaf, code);
                int sx, sy, sz;
                decode_shift(code, sx, sy, sz);
                off = make_float4((float)sx * A.L[0], (float)sy * A.L[1], (float)sz * A.L[2], __int_as_float(first));
                if (first + cnt > gself) {
                    const float4 bl = __ldg(A.box8 + 2 * (int64_t)leaf), bh = __ldg(A.box8 + 2 * (int64_t)leaf + 1);
                    const float gx = fmaxf(fmaxf(bl.x + off.x - hi[0], lo[0] - bh.x - off.x), 0.f);
                    const float gy = fmaxf(fmaxf(bl.y + off.y - hi[1], lo[1] - bh.y - off.y), 0.f);
                    const float gz = fmaxf(fmaxf(bl.z + off.z - hi[2], lo[2] - bh.z - off.z), 0.f);
                    ek = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) < wcut;
                }
            }
            const unsigned em = __ballot_sync(0xffffffffu, ek);
            if (ek) {
                const int q = __popc(em & below);
                S.woff[q] = off;
                S.wcnt[q] = cnt;
            }
            const int nsurv = __popc(em);
            __syncwarp();
            // two surviving j-leaves per half-warp instance
            for (int q0 = 0; q0 < nsurv; q0 += 2) {
                float4 op = ip;
                int oidx = iidx;
                if (!lower) {
                    const int qe = q0 + ((lane - 16) >> 3), kk = lane & 7;
                    oidx = -1;
                    if (qe < nsurv && kk < S.wcnt[qe]) {
                        const float4 o = S.woff[qe];
                        oidx = __float_as_int(o.w) + kk;
                        op = __ldg(A.xm + oidx);
                        op.x += o.x; op.y += o.y; op.z += o.z;  // exact (O1)
                    }
                }
#pragma unroll 4
                for (int k = 0; k < 16; ++k) {
                    const int m = 16 | k;
                    const float px = __shfl_xor_sync(0xffffffffu, op.x, m);
                    const float py = __shfl_xor_sync(0xffffffffu, op.y, m);
                    const float pz = __shfl_xor_sync(0xffffffffu, op.z, m);
                    const float pm = __shfl_xor_sync(0xffffffffu, op.w, m);
                    const int pidx = __shfl_xor_sync(0xffffffffu, oidx, m);
                    // the pair (i = lower lane's particle, j = upper's) is owned here iff j > i
                    const bool own = oidx >= 0 && pidx >= 0 && (lower ? pidx > oidx : oidx > pidx);
                    const float dx = px - op.x, dy = py - op.y, dz = pz - op.z;  // exact (O1)
                    const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));  // O2 order
                    const float ri = rsqrtf(r2 + e2);
                    float p5 = fmaf(c5, r2, c4);
                    p5 = fmaf(p5, r2, c3);
                    p5 = fmaf(p5, r2, c2);
                    p5 = fmaf(p5, r2, c1);
                    p5 = fmaf(p5, r2, c0);
                    const float wv = (own && r2 < rc2) ? pm * fmaf(ri * ri, ri, -p5) : 0.f;
                    acc[0] = fmaf(wv, dx, acc[0]);  // force of the partner on this lane's particle
                    acc[1] = fmaf(wv, dy, acc[1]);
                    acc[2] = fmaf(wv, dz, acc[2]);
                }
                if (!lower) {  // j-side sums: once per j-particle and instance
                    if (oidx >= 0) red_add_v4(A.acc + oidx, acc[0], acc[1], acc[2], 0.f);
                    acc[0] = acc[1] = acc[2] = 0.f;
                }
            }
            __syncwarp();
        }
        if (lower && iidx >= 0) red_add_v4(A.acc + iidx, acc[0], acc[1], acc[2], 0.f);
    }
}

// ------------------------------------------------------------ pipelined warp-independent variant
// With domain decomposition (A.partial) a pair with a ghost j is evaluated by i's group
// whatever j's index (the ghost has no group here) and its reaction is dropped (j's own
// rank evaluates the pair for j).
// Per warp a two-deep software pipeline of async copies (cp.async, no registers held): the
// entry cull is precomputed by the list build as one bit per (entry, i-group) (k_entry_masks:
// box test + Newton-3 / ghost rule), so the warp scans its row's mask bytes four entries per
// lane, queues the surviving entries, and streams chunks of 32 of them — the packed entries
// of chunk c+2 and the particles of chunk c+1 are in flight while chunk c is culled per
// particle and evaluated from shared memory.
namespace symp {
constexpr int G = 16, RING = 64, NW = 4, QCAP = 256;
// CAPL: the chunk size, surviving j-leaves whose particles are staged in shared memory per chunk
// (the queued chunks are full: a chunk larger than CAPL read a third of its leaves from L2)
template <int CAPL>
struct WarpSm {
    int2 ec[2][CAPL];           // packed list entries of two chunks of surviving entries
    int sq[QCAP];               // queue of surviving entry indices (mask scan)
    float4 pp[2][CAPL * JMAX];  // particles of the first CAPL leaves of two chunks
    float4 woff[2][CAPL];       // chunk entries: shift offset, first | (count - 1) << 29 (w)
    float4 wpos[RING];
    int widx[RING];
    float2 inx[G / 2], iny[G / 2], inz[G / 2], im[G / 2];
};
constexpr int SHIFT_BYTES = 27 * 16;  // per-CTA table of the 27 periodic offsets (shift code -> float4)
}  // namespace symp

// The benchmarked gravity kernel (crk_params.symmetric & 1, grav_kernel 0).  COUNT: the
// same work items, culls, ownership and ring with an integer payload — each evaluated pair
// that passes the O2 predicate adds 1 to both particles' counters (i-side in registers,
// reactions by red.global.add.s32) — so crk_count_pairs checks the coverage of exactly the
// kernel the bench times (SPEC.md:374-382 integer-payload audit, PAPER.md:418 pair symmetry).
template <bool PARTIAL, bool COUNT, int CAPL, int MINB>
__global__ void __launch_bounds__(symp::NW * 32, MINB) grav_pipe_kernel(const GravSymArgs A) {
    using namespace symp;
    using WS = WarpSm<CAPL>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    float4* shift_tab = reinterpret_cast<float4*>(smem_raw);
    WS& S = reinterpret_cast<WS*>(smem_raw + SHIFT_BYTES)[warp];
    const float wcut = A.wcut;
    const float rc2 = A.rcut2, e2 = A.eps2;
    const unsigned below = (1u << lane) - 1u;
    const float4* __restrict__ xm = A.xm;
    if (threadIdx.x < 27) {
        const int code = threadIdx.x;
        shift_tab[code] = make_float4((float)(code % 3 - 1) * A.L[0], (float)((code / 3) % 3 - 1) * A.L[1],
                                      (float)(code / 9 - 1) * A.L[2], 0.f);
    }
    __syncthreads();

    while (true) {
        int w = 0;
        if (lane == 0) w = atomicAdd(A.work, 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= A.nitems) break;
        const int a = w >> A.lsplit;
        const int gbit = w & (A.split - 1);  // the group's bit in the entry masks
        const int icount = __ldg(A.icount + a);
        const int ibase = gbit * G;
        if (ibase >= icount) continue;
        const int gself = __ldg(A.ifirst + a) + ibase;
        const int ng = min(G, icount - ibase);
        const int rbeg = __ldg(A.row_off + a), rend = __ldg(A.row_end + a);

        // mask scan: queue the row's entries whose bit gbit is set, in row order, until at least
        // CAPL wait or the row is exhausted (lane l reads the mask bytes of entries es + 4l .. + 3)
        int es = rbeg & ~3, qw = 0, qr = 0;
        auto refill = [&]() {
            while (qw - qr < CAPL && es < rend) {
                const int e = es + 4 * lane;
                uint32_t sel = 0;
                if (e < rend) {
                    const uint32_t wv = __ldg(reinterpret_cast<const uint32_t*>(A.gmask) + (e >> 2));
                    const uint32_t t = (wv >> gbit) & 0x01010101u;
                    sel = (t | (t >> 7) | (t >> 14) | (t >> 21)) & 0xfu;
                    if (e < rbeg) sel &= 0xfu << (rbeg - e);
                    if (rend - e < 4) sel &= (1u << (rend - e)) - 1u;
                }
                const int cnt = __popc(sel);
                const unsigned b0 = __ballot_sync(0xffffffffu, cnt & 1), b1 = __ballot_sync(0xffffffffu, cnt & 2),
                               b2 = __ballot_sync(0xffffffffu, cnt & 4);
                int pos = qw + __popc(b0 & below) + 2 * __popc(b1 & below) + 4 * __popc(b2 & below);
                while (sel) {
                    S.sq[pos & (QCAP - 1)] = e + __ffs(sel) - 1;
                    sel &= sel - 1;
                    ++pos;
                }
                qw += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
                es += 128;
            }
            __syncwarp();
        };
        // the next <= CAPL queued entries: their packed records -> ec[buf]
        auto issue_chunk = [&](int buf) {
            refill();
            const int n = min(CAPL, qw - qr);
            if (lane < n) cp_async8(&S.ec[buf][lane], A.erec + S.sq[(qr + lane) & (QCAP - 1)]);
            cp_async_commit();
            qr += n;
            return n;
        };

        float lo[3], hi[3];  // the group's box (nlh: (-lo, -hi) per axis, packed for the particle cull)
        {
            const bool iv = lane < ng;
            float4 p = make_float4(-1e18f, -1e18f, -1e18f, 0.f);
            if (iv) p = __ldg(xm + gself + lane);
            if (lane < G) {
                const int k = 2 * (lane % (G / 2)) + lane / (G / 2);
                reinterpret_cast<float*>(S.inx)[k] = -p.x;
                reinterpret_cast<float*>(S.iny)[k] = -p.y;
                reinterpret_cast<float*>(S.inz)[k] = -p.z;
                reinterpret_cast<float*>(S.im)[k] = p.w;
            }
            lo[0] = warp_min(iv ? p.x : INFINITY);
            lo[1] = warp_min(iv ? p.y : INFINITY);
            lo[2] = warp_min(iv ? p.z : INFINITY);
            hi[0] = warp_max(iv ? p.x : -INFINITY);
            hi[1] = warp_max(iv ? p.y : -INFINITY);
            hi[2] = warp_max(iv ? p.z : -INFINITY);
        }
        const float2 nlh[3] = {make_float2(-lo[0], -hi[0]), make_float2(-lo[1], -hi[1]), make_float2(-lo[2], -hi[2])};
        int n0 = issue_chunk(0), n1 = issue_chunk(1), n2 = 0;  // entries of chunks c, c + 1, c + 2

        // chunk entries landed in ec[buf]: shift offsets and the lane's leaf's particle copies
        // (all JMAX slots: xm is padded, members beyond the count are masked by the particle cull)
        auto decode = [&](int buf, int n) {
            if (lane < n) {
                const int2 r = S.ec[buf][lane];
                float4 off = shift_tab[(unsigned)r.y >> 26];
                off.w = __int_as_float(r.x);  // first | (count - 1) << 29
                S.woff[buf][lane] = off;
                if (lane < CAPL) {
                    const float4* src = xm + (r.x & 0x1fffffff);
#pragma unroll
                    for (int m = 0; m < JMAX; ++m) cp_async16(&S.pp[buf][lane * JMAX + m], src + m);
                }
            }
            cp_async_commit();
        };
        cp_async_wait<1>();  // entries(0)
        __syncwarp();
        decode(0, n0);

        // i-side sums, packed: component .x is i = k, .y is i = k + G/2
        float2 ax[G / 2], ay[G / 2], az[G / 2];
        int2 ci[COUNT ? G / 2 : 1];
#pragma unroll
        for (int k = 0; k < G / 2; ++k) ax[k] = ay[k] = az[k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < (COUNT ? G / 2 : 1); ++k) ci[k] = make_int2(0, 0);

        auto eval_step = [&](int r0, int n) {
            float4 jp = make_float4(1e18f, 1e18f, 1e18f, 0.f);
            int j = 0;
            if (lane < n) {
                const int s = (r0 + lane) & (RING - 1);
                jp = S.wpos[s];
                j = S.widx[s];
            }
            const bool jown = j >= gself && j < gself + ng;  // own group: the i-side half is counted
            const float2 jx = make_float2(jp.x, jp.x), jy = make_float2(jp.y, jp.y), jz = make_float2(jp.z, jp.z);
            if constexpr (COUNT) {
                // O2 membership, both directions; the pair (i, i) of a survivor in its own group is
                // not a pair.  i-side only when j is outside the group (met from both sides inside).
                int bj = 0;
#pragma unroll
                for (int k = 0; k < G / 2; ++k) {
                    const float2 dx = __fadd2_rn(jx, S.inx[k]);
                    const float2 dy = __fadd2_rn(jy, S.iny[k]);
                    const float2 dz = __fadd2_rn(jz, S.inz[k]);
                    const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
                    const bool in0 = lane < n && r2.x < rc2 && j != gself + k;
                    const bool in1 = lane < n && r2.y < rc2 && j != gself + k + G / 2;
                    ci[k].x += (in0 && !jown) ? 1 : 0;
                    ci[k].y += (in1 && !jown) ? 1 : 0;
                    bj += (in0 ? 1 : 0) + (in1 ? 1 : 0);
                }
                if (lane < n && (!PARTIAL || j >= 0) && bj) atomicAdd(A.cnt + j, bj);
            } else {
                const float mj = jown ? 0.f : jp.w;
                const float2 mj2 = make_float2(mj, mj), e22 = make_float2(e2, e2);
                const float2 n0 = make_float2(A.ne[0], A.ne[0]), n1 = make_float2(A.ne[1], A.ne[1]);
                const float2 n2 = make_float2(A.ne[2], A.ne[2]), n3 = make_float2(A.ne[3], A.ne[3]);
                const float2 n4 = make_float2(A.ne[4], A.ne[4]), n5 = make_float2(A.ne[5], A.ne[5]);
                const float rce = A.rce;
                float2 bx = make_float2(0.f, 0.f), by = bx, bz = bx;
#pragma unroll
                for (int k = 0; k < G / 2; ++k) {
                    const float2 dx = __fadd2_rn(jx, S.inx[k]);  // x_j - x_i, exact (O1)
                    const float2 dy = __fadd2_rn(jy, S.iny[k]);
                    const float2 dz = __fadd2_rn(jz, S.inz[k]);
                    // t = s + eps2, accumulated from eps2 (the force's cutoff t < rce; see ne, rce)
                    const float2 re = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, e22)));
                    const float2 ri = make_float2(rsqrtf(re.x), rsqrtf(re.y));
                    const float2 ri2 = __fmul2_rn(ri, ri);
                    float2 np5 = __ffma2_rn(n5, re, n4);  // -P5(t - eps2)
                    np5 = __ffma2_rn(np5, re, n3);
                    np5 = __ffma2_rn(np5, re, n2);
                    np5 = __ffma2_rn(np5, re, n1);
                    np5 = __ffma2_rn(np5, re, n0);
                    float2 wv = __ffma2_rn(ri2, ri, np5);  // t^-3/2 - P5(s)
                    wv.x = re.x < rce ? wv.x : 0.f;
                    wv.y = re.y < rce ? wv.y : 0.f;
                    const float2 wi = __fmul2_rn(mj2, wv);  // i-side: a_i += m_j w x_ji
                    ax[k] = __ffma2_rn(wi, dx, ax[k]);
                    ay[k] = __ffma2_rn(wi, dy, ay[k]);
                    az[k] = __ffma2_rn(wi, dz, az[k]);
                    const float2 wj = __fmul2_rn(S.im[k], wv);  // j-side: a_j -= m_i w x_ji
                    bx = __ffma2_rn(wj, dx, bx);
                    by = __ffma2_rn(wj, dy, by);
                    bz = __ffma2_rn(wj, dz, bz);
                }
                if (lane < n && (!PARTIAL || j >= 0))
                    red_add_v4(A.acc + j, -(bx.x + bx.y), -(by.x + by.y), -(bz.x + bz.y), 0.f);
            }
        };

        int wr = 0, rd = 0;
        for (int c = 0; n0 > 0; ++c) {
            const int b = c & 1;
            n2 = issue_chunk(b);  // chunk c + 2 into ec[b]: chunk c's entries were decoded
            cp_async_wait<2>();   // entries(c + 1)
            __syncwarp();
            decode(b ^ 1, n1);    // its particles go to pp[b ^ 1] (chunk c - 1's, consumed)
            cp_async_wait<2>();   // particles(c)
            __syncwarp();
            // particle cull of chunk c from shared memory, then evaluation:
            // lane -> (surviving entry q0 + lane / JMAX, member lane % JMAX)
            const int ns = n0;
            const int kk = lane % JMAX;
            const uint32_t ring_pos = opaque_u32(smem_u32(S.wpos)), ring_idx = ring_pos + (uint32_t)sizeof(S.wpos);
            auto cull_iter = [&](int q0) {
                const int q = q0 + lane / JMAX;
                const bool qv = q < ns;
                const int qc = qv ? q : 0;
                const float4 o = S.woff[b][qc];
                const int fc = __float_as_int(o.w);
                int j = (fc & 0x1fffffff) + kk;
                float4 p = S.pp[b][qc * JMAX + kk];
                bool keep = qv && kk <= (int)((unsigned)fc >> 29);
                if (PARTIAL && keep && !grav_owned(A, p.x, p.y, p.z)) j = -1 - j;  // ghost: no reaction
                const float2 pxy = __fadd2_rn(make_float2(p.x, p.y), make_float2(o.x, o.y));  // exact (O1)
                p.x = pxy.x; p.y = pxy.y; p.z += o.z;
                // box_dist2 packed: (p - lo, p - hi) per axis; max(-(p - lo), p - hi, 0) = max(lo - p, p - hi, 0)
                // exactly (fl(b - a) = -fl(a - b)), so the cull set is box_dist2's
                const float2 ux = __fadd2_rn(make_float2(p.x, p.x), nlh[0]);
                const float2 uy = __fadd2_rn(make_float2(p.y, p.y), nlh[1]);
                const float2 uz = __fadd2_rn(make_float2(p.z, p.z), nlh[2]);
                const float gx = fmaxf(fmaxf(-ux.x, ux.y), 0.f), gy = fmaxf(fmaxf(-uy.x, uy.y), 0.f);
                const float gz = fmaxf(fmaxf(-uz.x, uz.y), 0.f);
                const float d2 = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
                keep = keep & (j >= gself || (PARTIAL && j < 0)) & (d2 < wcut);
                const unsigned msk = __ballot_sync(0xffffffffu, keep);
                const uint32_t t = (uint32_t)(wr + __popc(msk & below)) & (RING - 1);
                if (keep) {
                    sts128(ring_pos + 16u * t, p);
                    sts32(ring_idx + 4u * t, j);
                }
                wr += __popc(msk);
                __syncwarp();
                if (wr - rd >= 32) {
                    eval_step(rd, 32);
                    rd += 32;
                    __syncwarp();
                }
            };
            for (int q0 = 0; q0 < ns; q0 += 32 / JMAX) cull_iter(q0);
            __syncwarp();
            n0 = n1;
            n1 = n2;
        }
        cp_async_wait<0>();
        if (wr > rd) eval_step(rd, wr - rd);
        if constexpr (COUNT) {
#pragma unroll
            for (int k = 0; k < G / 2; ++k) {
                const int t0 = __reduce_add_sync(0xffffffffu, ci[k].x), t1 = __reduce_add_sync(0xffffffffu, ci[k].y);
                if (lane == k && k < ng && t0) atomicAdd(A.cnt + gself + k, t0);
                if (lane == k + G / 2 && k + G / 2 < ng && t1) atomicAdd(A.cnt + gself + k + G / 2, t1);
            }
        } else {
            // transposed (reduce-scatter) sum of the 16 x 3 i-side values; lane l ends with i = l >> 1
            float v[3][G];
#pragma unroll
            for (int k = 0; k < G / 2; ++k) {
                v[0][k] = ax[k].x; v[0][k + G / 2] = ax[k].y;
                v[1][k] = ay[k].x; v[1][k + G / 2] = ay[k].y;
                v[2][k] = az[k].x; v[2][k + G / 2] = az[k].y;
            }
#pragma unroll
            for (int h = G / 2; h >= 1; h >>= 1) {
                const bool up = lane & (2 * h);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc)
#pragma unroll
                    for (int k = 0; k < h; ++k) {
                        const float send = up ? v[cc][k] : v[cc][k + h];
                        const float keep = up ? v[cc][k + h] : v[cc][k];
                        v[cc][k] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
                    }
            }
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) v[cc][0] += __shfl_xor_sync(0xffffffffu, v[cc][0], 1);
            if ((lane & 1) == 0 && (lane >> 1) < ng)
                red_add_v4(A.acc + gself + (lane >> 1), v[0][0], v[1][0], v[2][0], 0.f);
        }
        __syncwarp();
    }
}

// a = G acc (written to the caller), v += dt a
__global__ void k_grav_finish(int64_t n, const float4* __restrict__ acc, float G, float dt, float* ax, float* ay,
                              float* az, float* vx, float* vy, float* vz) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 q = acc[i];
    const float gx = G * q.x, gy = G * q.y, gz = G * q.z;
    if (ax) { ax[i] = gx; ay[i] = gy; az[i] = gz; }
    if (dt != 0.f) {
        vx[i] = fmaf(dt, gx, vx[i]);
        vy[i] = fmaf(dt, gy, vy[i]);
        vz[i] = fmaf(dt, gz, vz[i]);
    }
}


static RowView grav_rows(crk_ctx* c) {
    RowView rv;
    rv.ifirst = P<int32_t>(c->lfirst[0]);
    rv.icount = P<int32_t>(c->lcount[0]);
    rv.row_off = P<int32_t>(c->rowoff[0]);
    rv.row_end = P<int32_t>(c->rowend[0]);
    rv.erec = P<int2>(c->erec[0]);
    rv.box8 = P<float4>(c->lbox8[1]);
    for (int a = 0; a < 3; ++a) rv.L[a] = c->lay.L[a];
    return rv;
}

template <bool COUNT>
static crk_status launch_grav(crk_ctx* c, crk_particles* p, float dt, int32_t* cnt, cudaStream_t st) {
    GravPass<COUNT> g;
    g.xm = P<float4>(c->xm);
    g.jrows = g.xm;
    g.jpay = nullptr;
    g.rcut2 = c->prm.rcut2;
    g.eps2 = c->prm.eps2;
    g.G = c->prm.G;
    g.dt = dt;
    g.c0 = c->prm.poly[0]; g.c1 = c->prm.poly[1]; g.c2 = c->prm.poly[2];
    g.c3 = c->prm.poly[3]; g.c4 = c->prm.poly[4]; g.c5 = c->prm.poly[5];
    g.ax = p->ax; g.ay = p->ay; g.az = p->az;
    g.vx = p->vx; g.vy = p->vy; g.vz = p->vz;
    g.cnt = cnt;
    if (c->nleaf[0] == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, launch_pairs<GravPass<COUNT>, GRAV_NW, GRAV_G, 256, 2>(g, grav_rows(c), c->nleaf[0], st),
                       "gravity kernel"));
    c->launches++;
    return CRK_OK;
}

template <int NW, int ENT, int NB, int GI = 16, int MINB = 16 / NW>
static cudaError_t launch_grav_sym(crk_ctx* c, GravSymArgs& A, cudaStream_t st) {
    using Smem = typename symg::Cfg<NW, ENT, NB, GI>::Smem;
    const int smem = (int)sizeof(Smem);
    cudaError_t e = cudaFuncSetAttribute(grav_sym_kernel<NW, ENT, NB, GI, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    A.split = (c->prm.leaf_max_i + NW * GI - 1) / (NW * GI);
    A.nitems = (int)(c->nleaf[0] * A.split);
    int per_sm = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grav_sym_kernel<NW, ENT, NB, GI, MINB>, NW * 32, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    const int grid = (int)std::min<int64_t>(A.nitems, (int64_t)std::max(1, per_sm) * nsm);
    grav_sym_kernel<NW, ENT, NB, GI, MINB><<<grid, NW * 32, smem, st>>>(A);
    return cudaGetLastError();
}


static GravSymArgs grav_args(crk_ctx* c) {
    GravSymArgs A;
    A.xm = P<float4>(c->xm);
    A.gmask = P<uint8_t>(c->gmask);
    A.box8 = P<float4>(c->lbox8[1]);
    A.erec = P<int2>(c->erec[0]);
    A.row_off = P<int32_t>(c->rowoff[0]);
    A.row_end = P<int32_t>(c->rowend[0]);
    A.ifirst = P<int32_t>(c->lfirst[0]);
    A.icount = P<int32_t>(c->lcount[0]);
    A.acc = P<float4>(c->gacc);
    A.cnt = nullptr;
    for (int d = 0; d < 3; ++d) A.L[d] = c->lay.L[d];
    A.rcut2 = c->prm.rcut2;
    A.eps2 = c->prm.eps2;
    A.wcut = c->prm.rcut2 * CULL_SLACK;
    A.c0 = c->prm.poly[0]; A.c1 = c->prm.poly[1]; A.c2 = c->prm.poly[2];
    A.c3 = c->prm.poly[3]; A.c4 = c->prm.poly[4]; A.c5 = c->prm.poly[5];
    for (int k = 0; k < 6; ++k) A.nc[k] = -c->prm.poly[k];
    {  // P5(s) = sum_k c_k (t - eps2)^k = sum_m d_m t^m, d_m = sum_{k>=m} C(k, m) c_k (-eps2)^(k-m)
        const double e = c->prm.eps2;
        for (int m = 0; m < 6; ++m) {
            double d = 0.0, binom = 1.0, pw = 1.0;
            for (int k = m; k < 6; ++k) {
                d += binom * (double)c->prm.poly[k] * pw;
                binom = binom * (double)(k + 1) / (double)(k + 1 - m);
                pw *= -e;
            }
            A.ne[m] = (float)-d;
        }
        A.rce = c->prm.rcut2 + c->prm.eps2;
    }
    A.partial = c->lay.partial;
    A.inv_q = c->lay.inv_q;
    A.cs = c->lay.cs;
    for (int d = 0; d < 3; ++d) { A.dlo[d] = c->lay.dlo[d]; A.dhi[d] = c->lay.dhi[d]; }
    A.work = P<int>(c->work);
    A.split = (c->prm.leaf_max_i + symp::G - 1) / symp::G;
    A.lsplit = 0;
    while ((1 << A.lsplit) < A.split) ++A.lsplit;  // api.cu validates leaf_max_i in {16, 32, 64, 128}
    A.nitems = (int)(c->nleaf[0] * A.split);
    return A;
}

template <bool COUNT, int CAPL, int MINB>
static cudaError_t launch_pipe_cfg(crk_ctx* c, const GravSymArgs& A, cudaStream_t st) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    const int smem = symp::SHIFT_BYTES + (int)sizeof(symp::WarpSm<CAPL>) * symp::NW;
    auto k = A.partial ? grav_pipe_kernel<true, COUNT, CAPL, MINB> : grav_pipe_kernel<false, COUNT, CAPL, MINB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, symp::NW * 32, smem);
    k<<<nsm * std::max(1, per_sm), symp::NW * 32, smem, st>>>(A);
    return cudaGetLastError();
}

// the pipelined Newton-3 kernel in its launch configurations (crk_params.grav_kernel 0-2): the
// shared-memory leaf capacity per chunk and the resident CTAs per SM trade the staged share of
// the particle reads against occupancy
template <bool COUNT>
static cudaError_t launch_pipe(crk_ctx* c, const GravSymArgs& A, cudaStream_t st) {
    switch (c->prm.grav_kernel) {
    case 1: return launch_pipe_cfg<COUNT, 32, 4>(c, A, st);
    case 2: return launch_pipe_cfg<COUNT, 16, 6>(c, A, st);
    default: return launch_pipe_cfg<COUNT, 24, 5>(c, A, st);
    }
}

static bool pipe_kernel(crk_ctx* c) { return c->prm.grav_kernel <= 2; }

static crk_status gravity_sym(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    const int64_t n = c->n;
    CRK_TRY(grow(c, c->gacc, n * 16, st));
    CRK_TRY(cuda_check(c, zero_async(c->gacc.p, n * 16, st, c), "memset"));
    if (c->nleaf[0] > 0) {
        CRK_TRY(grow(c, c->work, 64, st));
        CRK_TRY(cuda_check(c, zero_async(c->work.p, 16, st, c), "memset"));
        GravSymArgs A = grav_args(c);
        cudaError_t e;
        switch (c->prm.grav_kernel) {
        case 6: {  // warp-independent without the copy pipeline
            int nsm = 0;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
            grav_warp_kernel<<<nsm * (16 / symw::NW), symw::NW * 32, 0, st>>>(A);
            e = cudaGetLastError();
            break;
        }
        case 7:  // CTA-staged rows (measured on c4, round 1: 24.6 ms)
            e = launch_grav_sym<8, 320, 1>(c, A, st);
            break;
        case 8: {  // the paper's half-warp shuffle algorithm (every pair evaluated once per direction)
            int nsm = 0;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
            grav_halfwarp_kernel<<<nsm * (16 / symh::NW), symh::NW * 32, 0, st>>>(A);
            e = cudaGetLastError();
            break;
        }
        default:  // pipelined warp-independent
            e = launch_pipe<false>(c, A, st);
            break;
        }
        if (e != cudaSuccess) return cuda_check(c, e, "gravity (symmetric) kernel");
        CRK_LAUNCHED(c, "gravity (symmetric) kernel");
    }
    k_grav_finish<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, P<float4>(c->gacc), c->prm.G, dt, p->ax, p->ay,
                                                                p->az, p->vx, p->vy, p->vz);
    CRK_LAUNCHED(c, "gravity finish");
    return CRK_OK;
}

crk_status gravity_kick(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    if (dt != 0.f && (!p->vx || !p->vy || !p->vz)) return fail(c, CRK_EINVAL, "kick needs vx, vy, vz");
    if ((c->prm.symmetric & 1) && (!c->lay.partial || pipe_kernel(c))) return gravity_sym(c, p, dt, st);
    return launch_grav<false>(c, p, dt, nullptr, st);
}

// count mode of the kernel crk_gravity_kick runs: the pipelined Newton-3 kernel with an integer
// payload when it is the configured one, else the i-centric kernel
crk_status gravity_count(crk_ctx* c, crk_particles* p, int32_t* cnt, cudaStream_t st) {
    if ((c->prm.symmetric & 1) && pipe_kernel(c)) {
        if (c->nleaf[0] == 0) return CRK_OK;
        CRK_TRY(grow(c, c->work, 64, st));
        CRK_TRY(cuda_check(c, zero_async(c->work.p, 16, st, c), "memset"));
        GravSymArgs A = grav_args(c);
        A.cnt = cnt;
        CRK_TRY(cuda_check(c, launch_pipe<true>(c, A, st), "gravity count kernel"));
        CRK_LAUNCHED(c, "gravity count kernel");
        return CRK_OK;
    }
    return launch_grav<true>(c, p, 0.f, cnt, st);
}

}  // namespace crk
