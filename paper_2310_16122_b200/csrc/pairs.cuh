// pairs.cuh — the list-driven pair-kernel skeleton shared by every force pass.
//
// One CTA per i-leaf (a row of the CSR leaf-pair list).  The
// CTA walks its row in chunks: all threads stage the particles of the next CH/JMAX
// j-leaves (periodic shift applied, so every difference is exact, O1) into shared
// memory; each warp then culls the staged candidates against the bounding box of
// its own G i-particles (ballot + popc compaction) and copies the survivors'
// positions (plus a payload index) into a warp-private buffer, which it then
// evaluates with a 4x unrolled loop.  Lane l holds i-particle l % G and takes every
// (32/G)-th survivor — the paper's half-warp layout (Fig.
// half-warp-layout: lanes 0-15 / 16-31) generalised to 32/G j-slots, i-centric, with
// register accumulation and one shuffle reduction over the slots at the end: no
// atomics (SURVEY.md §7 "B200-idiomatic design").
#pragma once
#include "common.cuh"

namespace crk {

struct RowView {
    const int32_t* ifirst;
    const int32_t* icount;
    const int32_t* jfirst;
    const int32_t* jcount;
    const int32_t* row_off;
    const int32_t* col;
    const int8_t* shift;
    const float* jbbox;   // 6 floats per j-leaf (lo xyz, hi xyz)
    const float* jmaxh2;  // per j-leaf max H^2 (SYM passes)
    float L[3];
};

// Pass concept:
//   static constexpr int PAY;            payload float4 per staged j (after the position)
//   static constexpr bool SYM;           culling radius also uses j's H^2 (jpos.w)
//   static constexpr int UNROLL;         survivors per lane per loop iteration
//   struct I; struct Acc;
//   void init(Acc&); void load_i(int i, I&); float ix/iy/iz(const I&); float cut(const I&)
//   void stage(int j, float ox, float oy, float oz, float4& jp, float4* pay)
//   void pair(const I&, Acc&, const float4& jp, const float4* pay)
//   template<int G> void reduce(Acc&) ; void finish(int i, const I&, const Acc&)
// Passes without payload copy the survivors' float4 into the warp list (one LDS.128 per
// pair); passes with a payload keep a u16 index list (the payload stays in the tile).
template <class Pass, int NW, int G, int CH>
struct PairSmem {
    static constexpr bool COPY = Pass::PAY == 0;
    float4 jpos[CH];
    float4 jpay[COPY ? 1 : CH * Pass::PAY];
    float4 wpos[COPY ? NW : 1][COPY ? CH : 1];
    uint16_t widx[COPY ? 1 : NW][COPY ? 1 : CH];
    uint8_t went[NW][32];
    float4 elo[CH / JMAX], ehi[CH / JMAX];  // shifted j-leaf boxes (.w of elo: max H^2)
};

template <class Pass, int NW, int G, int CH, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) pair_kernel(const Pass pass, const RowView rv) {
    static_assert(32 % G == 0, "G must divide the warp");
    static_assert(CH % 32 == 0 && CH % JMAX == 0, "bad chunk");
    constexpr int S = 32 / G;
    constexpr bool HASPAY = Pass::PAY > 0;
    using SM = PairSmem<Pass, NW, G, CH>;
    __shared__ SM sm;

    const int a = blockIdx.x;
    const int ifirst = rv.ifirst[a];
    const int icount = rv.icount[a];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int il = lane % G;
    const int sl = lane / G;
    const int ibase = warp * G;
    const bool wactive = ibase < icount;
    const bool ivalid = ibase + il < icount;
    float4* wpos = sm.wpos[SM::COPY ? warp : 0];
    uint16_t* widx = sm.widx[SM::COPY ? 0 : warp];
    uint8_t* went = sm.went[warp];
    static_assert(CH / JMAX <= 32, "one lane per staged j-leaf");

    typename Pass::I is;
    typename Pass::Acc acc;
    pass.init(acc);
    float lo[3], hi[3], wcut = 0.f;
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

    const int rbeg = rv.row_off[a], rend = rv.row_off[a + 1];
    constexpr int EPC = CH / JMAX;  // entries per chunk
    // chunk c takes the row entries c, c + nch, c + 2 nch, ...: every chunk samples the
    // whole neighbourhood, so the warps' per-chunk work (and the barrier wait) balances
    const int nch = (rend - rbeg + EPC - 1) / EPC;
    for (int c = 0; c < nch; ++c) {
        const int nent = (rend - rbeg - c + nch - 1) / nch;  // entries in this chunk
        for (int t = threadIdx.x; t < CH; t += NW * 32) {
            const int m = t / JMAX;
            const int k = t % JMAX;
            const int e = rbeg + c + m * nch;
            bool ok = false;
            int j = 0, code = 13, b = 0;
            if (m < nent) {
                b = __ldg(rv.col + e);
                code = __ldg(rv.shift + e);
                if (k < __ldg(rv.jcount + b)) {
                    ok = true;
                    j = __ldg(rv.jfirst + b) + k;
                }
            }
            int sx, sy, sz;
            decode_shift(code, sx, sy, sz);
            const float ox = (float)sx * rv.L[0], oy = (float)sy * rv.L[1], oz = (float)sz * rv.L[2];
            if (ok) {
                pass.stage(j, ox, oy, oz, sm.jpos[t], sm.jpay + (HASPAY ? t * Pass::PAY : 0));
            } else {
                sm.jpos[t] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
            }
            if (k == 0 && m < nent) {
                const float* bb = rv.jbbox + 6 * (int64_t)b;
                sm.elo[m] = make_float4(__ldg(bb) + ox, __ldg(bb + 1) + oy, __ldg(bb + 2) + oz,
                                        Pass::SYM ? __ldg(rv.jmaxh2 + b) * CULL_SLACK : 0.f);
                sm.ehi[m] = make_float4(__ldg(bb + 3) + ox, __ldg(bb + 4) + oy, __ldg(bb + 5) + oz, 0.f);
            }
        }
        __syncthreads();
        if (wactive) {
            // (1) leaf-level prefilter: one lane per staged j-leaf, box-box distance
            bool ek = false;
            if (lane < nent) {
                const float4 bl = sm.elo[lane], bh = sm.ehi[lane];
                const float gx = fmaxf(fmaxf(bl.x - hi[0], lo[0] - bh.x), 0.f);
                const float gy = fmaxf(fmaxf(bl.y - hi[1], lo[1] - bh.y), 0.f);
                const float gz = fmaxf(fmaxf(bl.z - hi[2], lo[2] - bh.z), 0.f);
                const float d2 = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
                ek = d2 < (Pass::SYM ? fmaxf(wcut, bl.w) : wcut);
            }
            const unsigned em = __ballot_sync(0xffffffffu, ek);
            if (ek) went[__popc(em & ((1u << lane) - 1u))] = (uint8_t)lane;
            const int nsurv = __popc(em);
            __syncwarp();
            // (2) particle-level filter over the surviving leaves, 32/JMAX leaves per step
            int cnt = 0;
            for (int q0 = 0; q0 < nsurv; q0 += 32 / JMAX) {
                const int qe = q0 + lane / JMAX;
                const int t = (qe < nsurv ? went[qe] : 0) * JMAX + lane % JMAX;
                float4 p = sm.jpos[t];
                if (qe >= nsurv) p.x = INFINITY;
                const float d2 = box_dist2(p.x, p.y, p.z, lo, hi);
                const bool keep = d2 < (Pass::SYM ? fmaxf(wcut, p.w * CULL_SLACK) : wcut);
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int o = cnt + __popc(m & ((1u << lane) - 1u));
                    if (SM::COPY) wpos[o] = p;
                    else widx[o] = (uint16_t)t;
                }
                cnt += __popc(m);
            }
            __syncwarp();
            constexpr int U = Pass::UNROLL;
            int k = sl;
#pragma unroll 1
            for (; k + (U - 1) * S < cnt; k += U * S) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int kk = k + u * S;
                    if (SM::COPY) {
                        pass.pair(is, acc, wpos[kk], sm.jpay);
                    } else {
                        const int t = widx[kk];
                        pass.pair(is, acc, sm.jpos[t], sm.jpay + t * Pass::PAY);
                    }
                }
            }
#pragma unroll 1
            for (; k < cnt; k += S) {
                if (SM::COPY) {
                    pass.pair(is, acc, wpos[k], sm.jpay);
                } else {
                    const int t = widx[k];
                    pass.pair(is, acc, sm.jpos[t], sm.jpay + t * Pass::PAY);
                }
            }
        }
        __syncthreads();
    }
    if (wactive) {
        pass.template reduce<G>(acc);
        if (ivalid && sl == 0) pass.finish(ifirst + ibase + il, is, acc);
    }
}

}  // namespace crk
