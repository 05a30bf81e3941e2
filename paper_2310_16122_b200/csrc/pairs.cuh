// pairs.cuh — the list-driven i-centric pair-kernel skeleton shared by the force passes.
//
// One CTA per i-leaf (a row of the CSR leaf-pair list).  The CTA
// copies its whole row — each j-leaf's packed position rows, payload rows and padded
// bounding box — into shared memory with 1-D TMA bulk copies (cp.async.bulk completing
// on one mbarrier; rows longer than ENT entries take several rounds).  After that single
// wait every warp works on its own: a leaf-level prefilter (box-box distance to the
// bounding box of its G i-particles), a particle-level filter (ballot + popc compaction
// into a per-warp survivor ring) and the evaluation, in which lane l holds i-particle
// l % G and takes every (32/G)-th survivor — the paper's half-warp layout (PAPER.md:418,
// Fig. half-warp-layout: lanes 0-15 / 16-31) generalised to 32/G j-slots, i-centric,
// register accumulation and one shuffle reduction over the slots at the end: no atomics.
// Periodic shifts are added to the staged positions (exact, O1).
#pragma once
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace crk {

struct RowView {
    const int32_t* ifirst;
    const int32_t* icount;
    const int32_t* row_off;  // row a: entries [row_off[a], row_end[a])
    const int32_t* row_end;
    const int2* erec;     // packed entries (first | (count-1) << 29, leaf | shift << 26)
    const float4* box8;   // padded j-leaf boxes: (lo, max H^2), (hi, 0)
    float L[3];
    const int32_t* rows = nullptr;  // non-null: run only rows[0 .. *nrows) (list fallback), grid-strided
    const int32_t* nrows = nullptr;
    // row subset (crk_select_rows): 0 every row, 1 the rows whose lists reference no ghost, 2 the
    // others (rclass[a] = 1: row a's list holds a ghost j-leaf), so that a decomposed substep can
    // run the interior rows while the ghost exchange is in flight
    const uint8_t* rclass = nullptr;
    int rsel = 0;
};
__device__ __forceinline__ bool row_selected(const RowView& rv, int a) { return rv.rsel == 0 || rv.rclass[a] == rv.rsel - 1; }

// Per-particle neighbour lists of the gas passes: row-relative staging
// slots (entry index within the i-leaf's CSR row * JMAX + member), ascending, of every
// gas j (self included) with s32 < max(H_i^2, H_j^2) — the symmetric predicate, a
// superset of the gather predicate.  Written by the geometry pass, read by corrections,
// extras and accel/du-dt.  Rows whose lists overflow `cap` (or whose slots exceed 16
// bits) are flagged; those rows run the on-the-fly kernels instead.
struct ListView {
    uint16_t* nbr;     // [n_gas * cap]
    int32_t* ncnt;     // [n_gas]
    uint32_t* lflag;   // [n gas i-leaves]: 1 = lists incomplete, use the on-the-fly path
    int32_t* frows;    // compact list of the flagged rows ...
    int32_t* nfrows;   // ... and their number (zeroed before the build)
    int cap;
    int nrows;         // rows (gas i-leaves)
    int* work;         // row counter of the persistent list kernels (zeroed per launch)
    int gate = 0;      // 1: the kernel runs only if some row is flagged (*nfrows > 0)
};
template <int G>
__device__ __forceinline__ unsigned same_i_lanes(int il) {  // lanes l with l % G == il
    unsigned m = 0;
#pragma unroll
    for (int q = 0; q < 32 / G; ++q) m |= 1u << (il + G * q);
    return m;
}

// Pass concept:
//   static constexpr int PAY;      payload float4 per j particle (contiguous rows in jpay)
//   static constexpr bool SYM;     culling radius also uses j's H^2 (symmetric predicate)
//   static constexpr int UNROLL;   survivors per lane per loop iteration
//   const float4* jrows; const float4* jpay;   j position rows (x, y, z, w) / payload rows
//   struct I; struct Acc;
//   void init(Acc&); void load_i(int i, I&); float ix/iy/iz(const I&); float cut(const I&)
//   float jcut(const float4& jp)   (SYM only: j's H^2 from its staged row)
//   void pair(const I&, Acc&, const float4& jp, const float4* pay, int j)
//   template<int G> void reduce(Acc&) ; void finish(int i, const I&, const Acc&)
// passes that declare `static constexpr bool PAIR2 = true` provide pair2(): two survivors at once
template <class Pass, class = void>
struct has_pair2 : std::false_type {};
template <class Pass>
struct has_pair2<Pass, std::enable_if_t<Pass::PAIR2>> : std::true_type {};
// passes that declare `static constexpr int BATCH` (32 or 64) and provide `bool in(const I&, float4 jp)`
// are evaluated pair-compacted: each batch of ring survivors is first tested against every
// i-particle of the warp (cheap), and the lanes of i-particle il then share only its in-range
// survivors, so a warp step does full work on (nearly) every lane instead of idling on
// out-of-range pairs.
// passes that declare `static constexpr bool BUILD = true` build the neighbour lists
// (ListView) while they evaluate: bool pair_list(const I&, Acc&, float4 jp, int j) returns
// the symmetric predicate of the pair, and Acc has an int `nl` (list length so far)
template <class Pass, class = void>
struct is_build : std::false_type {};
template <class Pass>
struct is_build<Pass, std::enable_if_t<Pass::BUILD>> : std::true_type {};
template <class Pass, class = void>
struct batch_of : std::integral_constant<int, 0> {};
template <class Pass>
struct batch_of<Pass, std::enable_if_t<(Pass::BATCH > 0)>> : std::integral_constant<int, Pass::BATCH> {};

template <class Pass, int NW, int ENT>
struct PairSmem {
    static constexpr int RING = batch_of<Pass>::value > 32 ? 128 : 64;
    float4 raw[ENT * JMAX];
    float4 pay[Pass::PAY > 0 ? ENT * JMAX * Pass::PAY : 1];
    float4 ebox[ENT][2];
    float4 eoff[ENT];  // shift offset (x, y, z), first (w, as int)
    int ecnt[ENT];
    uint64_t bar;
    uint16_t went[NW][ENT];
    float4 rpos[NW][RING];     // survivors: shifted position
    uint16_t rslot[NW][RING];  // survivors: staged slot (payload, j index)
};

template <class Pass, int NW, int G, int ENT>
__device__ __forceinline__ void pair_row(const Pass& pass, const RowView& rv, PairSmem<Pass, NW, ENT>& sm, const int a,
                                         uint32_t& phase) {
    static_assert(32 % G == 0, "G must divide the warp");
    static_assert(ENT * JMAX <= 65536, "slot index is 16 bits");
    constexpr int S = 32 / G;
    using SM = PairSmem<Pass, NW, ENT>;
    constexpr int RING = SM::RING;
    const int ifirst = rv.ifirst[a];
    const int icount = rv.icount[a];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int il = lane % G;
    const int sl = lane / G;
    const int ibase = warp * G;
    const bool wactive = ibase < icount;
    const bool ivalid = ibase + il < icount;
    const int rbeg = rv.row_off[a], rend = rv.row_end[a];
    int rbase = 0;  // row-relative slot of the current round's first entry
    [[maybe_unused]] int lcap = 0;
    if constexpr (is_build<Pass>::value)  // slots are 16-bit: longer rows get no lists
        lcap = (rend - rbeg) * JMAX <= 65536 ? pass.lv.cap : 0;
    float4* rpos = sm.rpos[warp];
    uint16_t* rslot = sm.rslot[warp];
    uint16_t* went = sm.went[warp];

    typename Pass::I is;
    typename Pass::Acc acc;
    pass.init(acc);
    float lo[3] = {0.f, 0.f, 0.f}, hi[3] = {0.f, 0.f, 0.f}, wcut = 0.f;
    if (wactive) {
        pass.load_i(ifirst + ibase + (ivalid ? il : 0), is);
        const float px = pass.ix(is), py = pass.iy(is), pz = pass.iz(is);
        lo[0] = warp_min(ivalid ? px : INFINITY);
        lo[1] = warp_min(ivalid ? py : INFINITY);
        lo[2] = warp_min(ivalid ? pz : INFINITY);
        hi[0] = warp_max(ivalid ? px : -INFINITY);
        hi[1] = warp_max(ivalid ? py : -INFINITY);
        hi[2] = warp_max(ivalid ? pz : -INFINITY);
        wcut = warp_max(ivalid ? pass.cut(is) : 0.f) * CULL_SLACK;
    }

    constexpr int BATCH = batch_of<Pass>::value;
    constexpr int TRIG = BATCH > 32 ? BATCH : 32;  // ring fill that triggers an evaluation
    // evaluate ring survivors [rd, rd + n)
    auto eval = [&](int rd, int n) {
        constexpr int U = Pass::UNROLL;
        int k = sl;
        if constexpr (is_build<Pass>::value) {  // every (i, survivor) pair tested, lists appended
            const unsigned own = same_i_lanes<G>(il);
            const int64_t lbase = (int64_t)(ifirst + ibase + il) * lcap;
            const unsigned below = own & ((1u << lane) - 1u);
            uint16_t* const lp = pass.lv.nbr + lbase;
            int k0 = 0;
#pragma unroll 1
            for (; k0 + 2 * S <= n; k0 += 2 * S) {  // two survivors per lane (packed FP32)
                bool ok0 = false, ok1 = false;
                const int s0 = (rd + k0 + sl) & (RING - 1), s1 = (rd + k0 + S + sl) & (RING - 1);
                const int t0 = rslot[s0], t1 = rslot[s1];
                if (ivalid) pass.pair_list2(is, acc, rpos[s0], rpos[s1], ok0, ok1);
                const unsigned b0 = __ballot_sync(0xffffffffu, ok0), b1 = __ballot_sync(0xffffffffu, ok1);
                const int n0 = __popc(b0 & own);
                const int pos0 = acc.nl + __popc(b0 & below), pos1 = acc.nl + n0 + __popc(b1 & below);
                if (ok0 && pos0 < lcap) lp[pos0] = (uint16_t)(rbase + t0);
                if (ok1 && pos1 < lcap) lp[pos1] = (uint16_t)(rbase + t1);
                acc.nl += n0 + __popc(b1 & own);
            }
#pragma unroll 1
            for (; k0 < n; k0 += S) {
                const int kk = k0 + sl;
                bool ok = false;
                int t = 0;
                if (ivalid && kk < n) {
                    const int s = (rd + kk) & (RING - 1);
                    t = rslot[s];
                    ok = pass.pair_list(is, acc, rpos[s], __float_as_int(sm.eoff[t / JMAX].w) + t % JMAX);
                }
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                const int pos = acc.nl + __popc(b & below);
                if (ok && pos < lcap) lp[pos] = (uint16_t)(rbase + t);
                acc.nl += __popc(b & own);
            }
            return;
        } else if constexpr (BATCH > 0) {  // pair-compacted (n <= BATCH)
            using M = std::conditional_t<(BATCH > 32), unsigned long long, unsigned>;
            M m = 0;
            if (ivalid)
                for (; k < n; k += S)
                    if (pass.in(is, rpos[(rd + k) & (RING - 1)])) m |= (M)1 << k;
#pragma unroll
            for (int o = G; o < 32; o <<= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
            // in-range survivors of i-particle il, shared round-robin by its S lanes
#pragma unroll
            for (int q = 0; q < S - 1; ++q)
                if (q < sl) m &= m - 1;
#pragma unroll 1
            while (m) {
                const int kk = (BATCH > 32 ? __ffsll((long long)m) : __ffs((int)m)) - 1;
#pragma unroll
                for (int q = 0; q < S; ++q) m &= m - 1;
                const int s = (rd + kk) & (RING - 1);
                const int t = rslot[s];
                pass.pair(is, acc, rpos[s], sm.pay + t * Pass::PAY, __float_as_int(sm.eoff[t / JMAX].w) + t % JMAX);
            }
            return;
        } else if constexpr (has_pair2<Pass>::value) {  // two survivors per packed-FP32 evaluation
#pragma unroll 1
            for (; k + S < n; k += 2 * S) {
                const int s0 = (rd + k) & (RING - 1), s1 = (rd + k + S) & (RING - 1);
                const int t0 = rslot[s0], t1 = rslot[s1];
                pass.pair2(is, acc, rpos[s0], sm.pay + t0 * Pass::PAY, __float_as_int(sm.eoff[t0 / JMAX].w) + t0 % JMAX,
                           rpos[s1], sm.pay + t1 * Pass::PAY, __float_as_int(sm.eoff[t1 / JMAX].w) + t1 % JMAX);
            }
        } else {
#pragma unroll 1
            for (; k + (U - 1) * S < n; k += U * S) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int s = (rd + k + u * S) & (RING - 1);
                    const int t = rslot[s];
                    pass.pair(is, acc, rpos[s], sm.pay + t * Pass::PAY,
                              __float_as_int(sm.eoff[t / JMAX].w) + t % JMAX);
                }
            }
        }
#pragma unroll 1
        for (; k < n; k += S) {
            const int s = (rd + k) & (RING - 1);
            const int t = rslot[s];
            pass.pair(is, acc, rpos[s], sm.pay + t * Pass::PAY, __float_as_int(sm.eoff[t / JMAX].w) + t % JMAX);
        }
    };

    int wr = 0, rd = 0;
    for (int e0 = rbeg; e0 < rend; e0 += ENT) {
        const int nent = min(ENT, rend - e0);
        rbase = (e0 - rbeg) * JMAX;
        __syncthreads();  // barrier initialised / previous round consumed
        // entry t is issued by warp t % NW: the bulk copies of one warp are issued lane by lane
        // (uniform operands), so spreading the row over all warps shortens the issue chain NW-fold.
        // (Merging runs of contiguous full leaves into one copy, as gravity does, measured slower
        // here: the serial run-length scan sits on the critical path of a one-round row.)
        for (int t = lane * NW + warp; t < nent; t += NW * 32) {
            int first, count, leaf, code;
            unpack_entry(__ldg(rv.erec + e0 + t), first, count, leaf, code);
            int sx, sy, sz;
            decode_shift(code, sx, sy, sz);
            sm.eoff[t] = make_float4((float)sx * rv.L[0], (float)sy * rv.L[1], (float)sz * rv.L[2],
                                     __int_as_float(first));
            sm.ecnt[t] = count;
            const uint32_t pb = (uint32_t)count * 16u;
            mbar_expect_tx(&sm.bar, pb * (1 + Pass::PAY) + 32u);
            bulk_g2s(&sm.raw[t * JMAX], pass.jrows + first, pb, &sm.bar);
            if (Pass::PAY > 0)
                bulk_g2s(&sm.pay[t * JMAX * Pass::PAY], pass.jpay + (int64_t)first * Pass::PAY, pb * Pass::PAY,
                         &sm.bar);
            bulk_g2s(&sm.ebox[t][0], rv.box8 + 2 * (int64_t)leaf, 32u, &sm.bar);
        }
        __syncthreads();
        if (threadIdx.x == 0) mbar_arrive(&sm.bar);
        mbar_wait(&sm.bar, phase);
        phase ^= 1u;
        if (wactive) {
            // (1) leaf prefilter
            int nsurv = 0;
            for (int e = lane; e - lane < nent; e += 32) {
                bool ek = false;
                if (e < nent) {
                    const float4 o = sm.eoff[e];
                    const float4 bl = sm.ebox[e][0], bh = sm.ebox[e][1];
                    const float gx = fmaxf(fmaxf(bl.x + o.x - hi[0], lo[0] - bh.x - o.x), 0.f);
                    const float gy = fmaxf(fmaxf(bl.y + o.y - hi[1], lo[1] - bh.y - o.y), 0.f);
                    const float gz = fmaxf(fmaxf(bl.z + o.z - hi[2], lo[2] - bh.z - o.z), 0.f);
                    const float d2 = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
                    ek = d2 < (Pass::SYM ? fmaxf(wcut, bl.w * CULL_SLACK) : wcut);
                }
                const unsigned em = __ballot_sync(0xffffffffu, ek);
                if (ek) went[nsurv + __popc(em & ((1u << lane) - 1u))] = (uint16_t)e;
                nsurv += __popc(em);
            }
            __syncwarp();
            // (2) particle filter into the survivor ring, evaluation whenever >= 32 wait
            for (int q0 = 0; q0 < nsurv; q0 += 32 / JMAX) {
                const int qe = q0 + lane / JMAX;
                const int kk = lane % JMAX;
                const int e = went[qe < nsurv ? qe : 0];
                const float4 o = sm.eoff[e];
                const int t = e * JMAX + kk;
                float4 p = sm.raw[t];
                p.x += o.x; p.y += o.y; p.z += o.z;
                bool keep = qe < nsurv && kk < sm.ecnt[e];
                if (keep) {
                    const float d2 = box_dist2(p.x, p.y, p.z, lo, hi);
                    keep = d2 < (Pass::SYM ? fmaxf(wcut, pass.jcut(p) * CULL_SLACK) : wcut);
                }
                const unsigned msk = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int s = (wr + __popc(msk & ((1u << lane) - 1u))) & (RING - 1);
                    if constexpr (is_build<Pass>::value) p.w = pass.jcut(p);  // the list predicate's H_j^2, once
                    rpos[s] = p;
                    rslot[s] = (uint16_t)t;
                }
                wr += __popc(msk);
                __syncwarp();
                if (wr - rd >= TRIG) {
                    eval(rd, TRIG);
                    rd += TRIG;
                    __syncwarp();
                }
            }
            if (e0 + ENT < rend && wr > rd) {  // slots are restaged next round: flush the ring
                eval(rd, wr - rd);
                rd = wr;
                __syncwarp();
            }
        }
    }
    if (wactive) {
        if (wr > rd) eval(rd, wr - rd);
        pass.template reduce<G>(acc);
        if (ivalid && sl == 0) {
            pass.finish(ifirst + ibase + il, is, acc);
            if constexpr (is_build<Pass>::value) {
                pass.lv.ncnt[ifirst + ibase + il] = acc.nl;
                if (acc.nl > lcap && atomicExch(pass.lv.lflag + a, 1u) == 0u)
                    pass.lv.frows[atomicAdd(pass.lv.nfrows, 1)] = a;
            }
        }
    }
}

template <class Pass, int NW, int G, int ENT, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) pair_kernel(const Pass pass, const RowView rv) {
    using SM = PairSmem<Pass, NW, ENT>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar, 1);
        mbar_fence_init();
    }
    uint32_t phase = 0;
    if (!rv.rows) {
        if (row_selected(rv, blockIdx.x)) pair_row<Pass, NW, G, ENT>(pass, rv, sm, blockIdx.x, phase);
        return;
    }
    const int nrows = *rv.nrows;
    for (int w = blockIdx.x; w < nrows; w += gridDim.x)
        if (row_selected(rv, rv.rows[w])) pair_row<Pass, NW, G, ENT>(pass, rv, sm, rv.rows[w], phase);
}

// ---------------------------------------------------------------- list-driven consumer
// Same row staging (positions and payload rows only: no boxes, no culling); lane l holds
// i-particle l % G and walks every (32/G)-th entry of i's neighbour list, so every
// evaluated pair is in the symmetric predicate (the gather passes still apply their own
// s32 < H_i^2 select).  Rows flagged by the list builder exit here and run pair_kernel
// with RowView::rows = the builder's flagged-row list.
// IREC (passes that declare `static constexpr bool IREC = true`): the first round of a row
// also stages the row's i-particles' 9-float4 records (pass.grec), position rows and list
// lengths, so that a new row's i-data come from shared memory instead of dependent global
// loads at the start of every CTA
template <class Pass, class = void>
struct has_irec : std::false_type {};
template <class Pass>
struct has_irec<Pass, std::enable_if_t<Pass::IREC>> : std::true_type {};
constexpr int LIST_IMAX = 64;  // gas i-leaf <= 64
template <int PAY, int ENT, bool IREC = false>
struct ListSmem {
    float4 raw[ENT * JMAX];
    float4 pay[PAY > 0 ? ENT * JMAX * PAY : 1];
    float4 eoff[ENT];  // shift offset (x, y, z), first (w, as int)
    float4 irec[IREC ? LIST_IMAX * 9 : 1];
    float4 ipos[IREC ? LIST_IMAX : 1];
    int icnt[IREC ? LIST_IMAX + 8 : 1];
    uint64_t bar;
    int next;          // claimed row
};
struct IStage {  // i-data of a row staged with its first round (IREC)
    const float4* grec;
    const float4* gpos;
    const int32_t* ncnt;
    int ifirst, icount;
    const void* lsrc = nullptr;  // optional: a further contiguous block (the row's neighbour lists)
    void* ldst = nullptr;
    uint32_t lbytes = 0;         // multiple of 16
};

// all threads: stage row entries [e0, e0 + nent) — position rows (x, y, z, w) and PAY payload
// float4 per particle — then apply the periodic shifts in place (once per slot, exact, O1);
// returns with the round resident and visible to the CTA
template <int PAY, int NW, int ENT, bool IREC = false>
__device__ __forceinline__ void stage_list_round(ListSmem<PAY, ENT, IREC>& sm, const RowView& rv, const float4* jrows,
                                                 const float4* jpay, int e0, int nent, uint32_t& phase,
                                                 const IStage* ist = nullptr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // barrier initialised / previous round consumed
    if constexpr (IREC) {
        if (ist && threadIdx.x == NW * 32 - 1) {
            const int c0 = ist->ifirst & ~3, c1 = (ist->ifirst + ist->icount + 3) & ~3;  // 16-byte aligned cover
            mbar_expect_tx(&sm.bar, (uint32_t)ist->icount * 160u + (uint32_t)(c1 - c0) * 4u);
            bulk_g2s(sm.irec, ist->grec + (int64_t)ist->ifirst * 9, (uint32_t)ist->icount * 144u, &sm.bar);
            bulk_g2s(sm.ipos, ist->gpos + ist->ifirst, (uint32_t)ist->icount * 16u, &sm.bar);
            bulk_g2s(sm.icnt, ist->ncnt + c0, (uint32_t)(c1 - c0) * 4u, &sm.bar);
        }
    }
    if (ist && ist->lbytes && threadIdx.x == NW * 32 - 2) {
        mbar_expect_tx(&sm.bar, ist->lbytes);
        bulk_g2s(ist->ldst, ist->lsrc, ist->lbytes, &sm.bar);
    }
    for (int t = lane * NW + warp; t < nent; t += NW * 32) {
        int first, count, leaf, code;
        unpack_entry(__ldg(rv.erec + e0 + t), first, count, leaf, code);
        int sx, sy, sz;
        decode_shift(code, sx, sy, sz);
        sm.eoff[t] = make_float4((float)sx * rv.L[0], (float)sy * rv.L[1], (float)sz * rv.L[2], __int_as_float(first));
        const uint32_t pb = (uint32_t)count * 16u;
        mbar_expect_tx(&sm.bar, pb * (1 + PAY));
        bulk_g2s(&sm.raw[t * JMAX], jrows + first, pb, &sm.bar);
        if (PAY > 0) bulk_g2s(&sm.pay[t * JMAX * PAY], jpay + (int64_t)first * PAY, pb * PAY, &sm.bar);
    }
    __syncthreads();
    if (threadIdx.x == 0) mbar_arrive(&sm.bar);
    mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    for (int t = threadIdx.x; t < nent * JMAX; t += NW * 32) {
        const float4 o = sm.eoff[t / JMAX];
        if (o.x != 0.f || o.y != 0.f || o.z != 0.f) {
            float4 q = sm.raw[t];
            q.x += o.x; q.y += o.y; q.z += o.z;
            sm.raw[t] = q;
        }
    }
    fence_proxy_async_smem();  // generic writes before the next round's TMA overwrites
    __syncthreads();
}

// persistent CTAs claim rows from lv.work; returns the claimed row (>= nrows: done)
template <class SM>
__device__ __forceinline__ int claim_row(SM& sm, int* work) {
    if (threadIdx.x == 0) sm.next = atomicAdd(work, 1);
    __syncthreads();
    const int a = sm.next;
    __syncthreads();  // every thread has read `next` before it is claimed again
    return a;
}

// G i-particles per warp, S = 32/G lanes per i.  A CTA covers NW*G i-particles at a time and
// loops over the row's i-particles in NW*G-sized iterations (G = 8 with 8 warps: one iteration
// per gas i-leaf of <= 64).  A row that fits one staging round is staged once for all
// iterations; longer rows are restaged per iteration.
// SEL: honour the row subset (crk_select_rows); a separate instantiation, since the check alone
// cost the accel walk 0.23 ms on c4 (code generation of the row body)
// SL: the row's neighbour lists staged into shared memory with its first round (as list_kernel2);
// needs one i-iteration per row (NW * G >= the gas i-leaf size)
template <int PAY, int ENT, bool IREC>
__host__ __device__ constexpr int list_sl_off() { return (int)((sizeof(ListSmem<PAY, ENT, IREC>) + 127) / 128 * 128); }
template <class Pass, int NW, int G, int ENT, int MINB, bool SEL = false, bool SL = false>
__global__ void __launch_bounds__(NW * 32, MINB) list_kernel(const Pass pass, const RowView rv, const ListView lv) {
    static_assert(32 % G == 0, "G must divide the warp");
    static_assert(!SL || NW * G >= LIST_IMAX, "staged lists: one i-iteration per row");
    constexpr int S = 32 / G;
    constexpr bool IREC = has_irec<Pass>::value;
    using SM = ListSmem<Pass::PAY, ENT, IREC>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    uint16_t* const lst = reinterpret_cast<uint16_t*>(smem_raw + list_sl_off<Pass::PAY, ENT, IREC>());
    if (lv.gate && *lv.nfrows == 0) return;  // gated fallback: only when some row is flagged

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // runs of S consecutive lanes share one i: the S lanes read consecutive list entries,
    // usually consecutive staged slots, so their shared-memory loads fall in distinct banks
    const int il = lane / S;
    const int sl = lane % S;
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar, 1);
        mbar_fence_init();
    }
    uint32_t phase = 0;
    auto row = [&](const int a) {
        const int ifirst = rv.ifirst[a];
        const int icount = rv.icount[a];
        const int rbeg = rv.row_off[a], rend = rv.row_end[a];
        const bool one_round = rend - rbeg <= ENT;
        const int nit = (icount + NW * G - 1) / (NW * G);
        IStage ist;
        if constexpr (IREC) {
            ist.grec = pass.grec; ist.gpos = pass.gpos; ist.ncnt = lv.ncnt;
            ist.ifirst = ifirst; ist.icount = icount;
        }
        if constexpr (SL) {
            ist.lsrc = lv.nbr + (int64_t)ifirst * lv.cap;
            ist.ldst = lst;
            ist.lbytes = (uint32_t)(icount * lv.cap * (int)sizeof(uint16_t));
        }
        if (one_round)
            stage_list_round<Pass::PAY, NW, ENT, IREC>(sm, rv, pass.jrows, pass.jpay, rbeg, rend - rbeg, phase,
                                                        (IREC || SL) ? &ist : nullptr);
        for (int it = 0; it < nit; ++it) {
            const int ibase = (it * NW + warp) * G;
            const bool wactive = ibase < icount;
            const bool ivalid = ibase + il < icount;
            typename Pass::I is;
            typename Pass::Acc acc;
            pass.init(acc);
            const int ki = ifirst + ibase + (ivalid ? il : 0);
            int nl = 0;
            if (wactive) {
                bool staged = false;
                if constexpr (IREC) {
                    if (one_round) {  // i-data from the staged copy
                        const int ii = ki - ifirst;
                        pass.load_i_staged(ki, sm.ipos[ii], &sm.irec[ii * 9], is);
                        nl = ivalid ? sm.icnt[ii + (ifirst & 3)] : 0;
                        staged = true;
                    }
                }
                if (!staged) {
                    pass.load_i(ki, is);
                    if (ivalid) nl = lv.ncnt[ki];
                }
            }
            const uint16_t* lp = lv.nbr + (int64_t)ki * lv.cap + sl;  // this lane's next list entry
            const uint16_t* const lend = lv.nbr + (int64_t)ki * lv.cap + nl;
            // SL: the same entries in the staged copy of the row's lists (offset ls from the start)
            const uint16_t* const lsm = lst + (ki - ifirst) * lv.cap;
            int ls = sl;
            auto next = [&]() -> int {
                if constexpr (SL) return ls < nl ? (int)lsm[ls] : 0x7fffffff;
                return lp < lend ? (int)*lp : 0x7fffffff;
            };
            int tn = (!SL || one_round) ? next() : 0x7fffffff;  // next slot of this lane
            for (int e0 = rbeg; e0 < rend; e0 += ENT) {
                const int nent = min(ENT, rend - e0);
                if (!one_round) {
                    stage_list_round<Pass::PAY, NW, ENT, IREC>(sm, rv, pass.jrows, pass.jpay, e0, nent, phase,
                                                                (SL && e0 == rbeg) ? &ist : nullptr);
                    if (SL && e0 == rbeg) tn = next();  // the lists landed with the first round
                }
                if (wactive) {
                    const int rs = (e0 - rbeg) * JMAX, re = rs + nent * JMAX;
#pragma unroll 1
                    while (__any_sync(0xffffffffu, tn < re)) {
                        if (tn < re) {
                            const int tl = tn - rs;
                            const float4 jp = sm.raw[tl];
                            lp += S;
                            ls += S;
                            tn = next();
                            pass.pair(is, acc, jp, sm.pay + tl * Pass::PAY,
                                      __float_as_int(sm.eoff[tl / JMAX].w) + tl % JMAX);
                        }
                    }
                }
            }
            if (wactive) {
                pass.template reduce<-S>(acc);
                if (ivalid && sl == 0) pass.finish(ki, is, acc);
            }
        }
    };
    if (!lv.gate) {  // one CTA per row (measured faster than claiming rows: the hardware
        if (!lv.lflag[blockIdx.x] && (!SEL || row_selected(rv, blockIdx.x))) row(blockIdx.x);  // overlaps a new CTA's staging)
        return;
    }
    while (true) {  // gated (rarely run) launches are persistent so that an idle launch is cheap
        const int a = claim_row(sm, lv.work);
        if (a >= lv.nrows) break;
        if (!lv.lflag[a] && (!SEL || row_selected(rv, a))) row(a);
    }
}

// Two list walks per row in one kernel: pass A over i's whole list, A's epilogue, then pass
// B (whose load_i may read what A's epilogue wrote for the same i: the same warp, ordered by
// __syncwarp).  The staged rows carry B's payload; a row that fits one round is staged once
// for both walks, longer rows are staged again for B.  Used to fuse Corrections and Extras:
// Extras needs only i's own coefficients, which Corrections has just produced.
// SL: the row's neighbour lists (consecutive gas ranks: one contiguous block of icount * cap
// 16-bit entries) are staged into shared memory with the first round, so that the walks read
// their next entry from shared memory instead of a dependent global load per pair
template <int PAY, int ENT>
__host__ __device__ constexpr int list2_sl_off() { return (int)((sizeof(ListSmem<PAY, ENT>) + 127) / 128 * 128); }
template <class PA, class PB, int NW, int G, int ENT, int MINB, bool SL = false>
__global__ void __launch_bounds__(NW * 32, MINB) list_kernel2(const PA pa, const PB pb, const RowView rv,
                                                              const ListView lv) {
    static_assert(32 % G == 0, "G must divide the warp");
    static_assert(PA::PAY == 0, "pass A reads positions only");
    constexpr int S = 32 / G;
    using SM = ListSmem<PB::PAY, ENT>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    uint16_t* const lst = reinterpret_cast<uint16_t*>(smem_raw + list2_sl_off<PB::PAY, ENT>());
    const int a = blockIdx.x;
    if (lv.lflag[a] || !row_selected(rv, a)) return;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int il = lane / S;
    const int sl = lane % S;
    const int ibase = warp * G;
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar, 1);
        mbar_fence_init();
    }
    uint32_t phase = 0;
    const int ifirst = rv.ifirst[a];
    const int icount = rv.icount[a];
    const bool wactive = ibase < icount;
    const bool ivalid = ibase + il < icount;
    const int rbeg = rv.row_off[a], rend = rv.row_end[a];
    const int ki = ifirst + ibase + (ivalid ? il : 0);
    const int nl = (wactive && ivalid) ? lv.ncnt[ki] : 0;
    const uint16_t* const lbeg = lv.nbr + (int64_t)ki * lv.cap;
    const uint16_t* const lsm = lst + (ibase + il) * lv.cap;  // SL: i's staged list
    const bool one_round = rend - rbeg <= ENT;
    IStage ist;
    if constexpr (SL) {
        ist.lsrc = lv.nbr + (int64_t)ifirst * lv.cap;
        ist.ldst = lst;
        ist.lbytes = (uint32_t)(icount * lv.cap * (int)sizeof(uint16_t));
    }
    auto lget = [&](int q) -> int { return SL ? (int)lsm[q] : (int)__ldg(lbeg + q); };

    // walk this lane's entries of round [e0, e0 + nent) with pass P (one entry per iteration:
    // two per iteration with a far sentinel measured slower here, 11.1 vs 10.5 ms on c4 — the
    // 80 registers it needs cost a resident CTA per SM)
    auto walk = [&](const auto& P, auto& is, auto& acc, int& lp, int& tn, int e0, int nent) {
        const int rs = (e0 - rbeg) * JMAX, re = rs + nent * JMAX;
#pragma unroll 1
        while (__any_sync(0xffffffffu, tn < re)) {
            if (tn < re) {
                const int tl = tn - rs;
                const float4 jp = sm.raw[tl];
                lp += S;
                tn = lp < nl ? lget(lp) : 0x7fffffff;
                P.pair(is, acc, jp, sm.pay + tl * PB::PAY, __float_as_int(sm.eoff[tl / JMAX].w) + tl % JMAX);
            }
        }
    };
    {  // pass A
        typename PA::I is;
        typename PA::Acc acc;
        pa.init(acc);
        if (wactive) pa.load_i(ki, is);
        int lp = sl;
        int tn = (!SL && lp < nl) ? (int)__ldg(lbeg + lp) : 0x7fffffff;
        for (int e0 = rbeg; e0 < rend; e0 += ENT) {
            const int nent = min(ENT, rend - e0);
            stage_list_round<PB::PAY, NW, ENT>(sm, rv, pb.jrows, pb.jpay, e0, nent, phase,
                                               (SL && e0 == rbeg) ? &ist : nullptr);
            if (SL && e0 == rbeg) tn = lp < nl ? lget(lp) : 0x7fffffff;  // the lists landed with the round
            if (wactive) walk(pa, is, acc, lp, tn, e0, nent);
        }
        if (wactive) {
            pa.template reduce<-S>(acc);
            if (ivalid && sl == 0) pa.finish(ki, is, acc);
        }
    }
    __syncwarp();
    {  // pass B
        typename PB::I is;
        typename PB::Acc acc;
        pb.init(acc);
        if (wactive) pb.load_i(ki, is);
        int lp = sl;
        int tn = lp < nl ? lget(lp) : 0x7fffffff;
        for (int e0 = rbeg; e0 < rend; e0 += ENT) {
            const int nent = min(ENT, rend - e0);
            if (!one_round) stage_list_round<PB::PAY, NW, ENT>(sm, rv, pb.jrows, pb.jpay, e0, nent, phase);
            if (wactive) walk(pb, is, acc, lp, tn, e0, nent);
        }
        if (wactive) {
            pb.template reduce<-S>(acc);
            if (ivalid && sl == 0) pb.finish(ki, is, acc);
        }
    }
}

template <class PA, class PB, int NW, int G, int ENT, int MINB>
inline cudaError_t launch_list2(const PA& pa, const PB& pb, const RowView& rv, const ListView& lv, cudaStream_t st,
                                bool stage_lists = false) {
    // staged lists: one gas i-leaf's lists (<= NW * G lists of cap 16-bit entries, 16-byte multiples)
    const bool sl = stage_lists && lv.cap % 8 == 0;
    const int smem = sl ? list2_sl_off<PB::PAY, ENT>() + NW * G * lv.cap * (int)sizeof(uint16_t)
                        : (int)sizeof(ListSmem<PB::PAY, ENT>);
    auto k = sl ? list_kernel2<PA, PB, NW, G, ENT, MINB, true> : list_kernel2<PA, PB, NW, G, ENT, MINB, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (lv.nrows <= 0) return cudaSuccess;
    k<<<lv.nrows, NW * 32, smem, st>>>(pa, pb, rv, lv);
    return cudaGetLastError();
}

// persistent grid for a list-driven kernel: as many CTAs as fit, each claiming rows
template <class K>
inline int persistent_grid(K kernel, int threads, int smem, int64_t nrows) {
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>(nrows, (int64_t)std::max(1, per_sm) * nsm));
}

template <class Pass, int NW, int G, int ENT, int MINB, bool SL = false>
inline cudaError_t launch_list(const Pass& pass, const RowView& rv, const ListView& lv, cudaStream_t st) {
    constexpr bool IREC = has_irec<Pass>::value;
    const int smem = SL ? list_sl_off<Pass::PAY, ENT, IREC>() + NW * G * lv.cap * (int)sizeof(uint16_t)
                        : (int)sizeof(ListSmem<Pass::PAY, ENT, IREC>);
    auto k = rv.rsel ? list_kernel<Pass, NW, G, ENT, MINB, true, SL> : list_kernel<Pass, NW, G, ENT, MINB, false, SL>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (lv.nrows <= 0) return cudaSuccess;
    if (lv.gate) {
        e = zero_async(lv.work, sizeof(int), st);
        if (e != cudaSuccess) return e;
    }
    k<<<lv.gate ? persistent_grid(k, NW * 32, smem, lv.nrows) : lv.nrows, NW * 32, smem, st>>>(pass, rv, lv);
    return cudaGetLastError();
}

template <class Pass, int NW, int G, int ENT, int MINB>
inline cudaError_t launch_pairs(const Pass& pass, const RowView& rv, int64_t nleaf, cudaStream_t st) {
    const int smem = (int)sizeof(PairSmem<Pass, NW, ENT>);
    cudaError_t e = cudaFuncSetAttribute(pair_kernel<Pass, NW, G, ENT, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // rows mode: a few CTAs per SM walk the (device-counted) row list
    const int64_t grid = rv.rows ? std::min<int64_t>(nleaf, 148 * MINB) : nleaf;
    if (grid <= 0) return cudaSuccess;
    pair_kernel<Pass, NW, G, ENT, MINB><<<(unsigned)grid, NW * 32, smem, st>>>(pass, rv);
    return cudaGetLastError();
}

}  // namespace crk
