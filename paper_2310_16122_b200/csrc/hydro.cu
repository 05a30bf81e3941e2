// hydro.cu — the five hot CRK-SPH kernels (timers upGeo, upCor,
// upBarEx, upBarAc/upBarDu at PAPER.md:503) as list-driven pair kernels over the gas
// leaves (formulas §8(c) O6-O9, readings in DESIGN.md §2).
//
// Gas state lives in the ctx in gas-rank order (gpos, gvel, gV, gcoef, grec) so that
// the j-tiles of every pass are contiguous; the caller's per-particle outputs are
// written at gas_idx[k] in each pass epilogue.

#include "pairs.cuh"

namespace crk {


struct HydCommon {
    const float4* gpos;      // (x, y, z, H)
    const int32_t* gas_idx;  // gas rank -> sorted position
};

__device__ __forceinline__ void load_pos(const float4* gpos, int k, float& x, float& y, float& z,
                                         float& H2, float& invH) {
    const float4 p = gpos[k];
    x = p.x; y = p.y; z = p.z;
    H2 = __fmul_rn(p.w, p.w);
    invH = 1.f / p.w;
}

// ---------------------------------------------------------------- packed FP32 helpers
// Two pairs per instruction with FFMA2 / FADD2 / FMUL2 (sm_100a): each op rounds per
// component exactly like its scalar form, so predicates and sums are unchanged.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 f2sel(bool px, bool py, float2 v) {
    return make_float2(px ? v.x : 0.f, py ? v.y : 0.f);
}
// Wendland C4 factors of two pairs: wt = (1-q)^6 (1+6q+35q^2/3), gt = -(56/3)(1-q)^5(1+5q)
__device__ __forceinline__ void wendland_t2(float2 s, float invH, float2& wt, float2& gt_h2) {
    const float2 r = make_float2(sqrtf(s.x), sqrtf(s.y));
    const float2 q = __fmul2_rn(r, f2(invH));
    const float2 t = make_float2(fmaxf(1.f - q.x, 0.f), fmaxf(1.f - q.y, 0.f));
    const float2 t2 = __fmul2_rn(t, t);
    const float2 t5 = __fmul2_rn(__fmul2_rn(t2, t2), t);
    wt = __fmul2_rn(__fmul2_rn(t5, t), __ffma2_rn(q, __ffma2_rn(q, f2(35.f / 3.f), f2(6.f)), f2(1.f)));
    gt_h2 = __fmul2_rn(__fmul2_rn(f2(-56.f / 3.f), t5), __ffma2_rn(f2(5.f), q, f2(1.f)));
}
__device__ __forceinline__ float2 s32_of2(float2 dx, float2 dy, float2 dz) {
    return __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
}

// ============================================================== a4 Geometry (upGeo)
// V_i = 1 / sum_{gas j, s32 < H_i^2, j incl. i} W(r_ij, H_i)
// LIST: also build the gas neighbour lists (pairs.cuh ListView): culling and list use the
// symmetric predicate s32 < max(H_i^2, H_j^2); V sums only the gather pairs.
template <bool COUNT, bool LIST = false>
struct GeoPass : HydCommon {
    static constexpr int PAY = 0;
    static constexpr bool SYM = LIST;
    static constexpr bool BUILD = LIST;
    ListView lv;
    static constexpr int UNROLL = 4;
    const float4* jrows;  // gpos
    const float4* jpay;
    float* gV;
    float4* gposV;        // out: (x, y, z, V) rows for the next passes
    float* Vout;
    int32_t* cnt;
    static constexpr bool PAIR2 = !COUNT;
    struct I { float x, y, z, H2, invH; int idx; };
    struct Acc { float2 w; int n, nl; };
    __device__ void init(Acc& a) const { a.w = make_float2(0.f, 0.f); a.n = 0; a.nl = 0; }
    __device__ void load_i(int k, I& s) const { load_pos(gpos, k, s.x, s.y, s.z, s.H2, s.invH); s.idx = k; }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I& s) const { return s.H2; }
    __device__ float jcut(const float4& jp) const { return __fmul_rn(jp.w, jp.w); }
    __device__ __forceinline__ bool pair_list(const I& s, Acc& a, const float4& jp, int) const {
        const float dx = jp.x - s.x, dy = jp.y - s.y, dz = jp.z - s.z;
        const float r2 = s32_of(dx, dy, dz);
        float wt, gt;
        wendland_t(r2, s.invH, wt, gt);
        a.w.x += r2 < s.H2 ? wt : 0.f;
        return r2 < fmaxf(s.H2, jp.w);  // (ring rows of the list build carry H_j^2, pairs.cuh)
    }
    __device__ __forceinline__ void pair_list2(const I& s, Acc& a, const float4& p0, const float4& p1, bool& ok0,
                                               bool& ok1) const {
        const float2 dx = make_float2(p0.x - s.x, p1.x - s.x), dy = make_float2(p0.y - s.y, p1.y - s.y),
                     dz = make_float2(p0.z - s.z, p1.z - s.z);
        const float2 r2 = s32_of2(dx, dy, dz);
        float2 wt, gt;
        wendland_t2(r2, s.invH, wt, gt);
        a.w = __fadd2_rn(a.w, f2sel(r2.x < s.H2, r2.y < s.H2, wt));
        ok0 = r2.x < fmaxf(s.H2, p0.w);
        ok1 = r2.y < fmaxf(s.H2, p1.w);
    }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4*, int j) const {
        const float dx = jp.x - s.x, dy = jp.y - s.y, dz = jp.z - s.z;
        const float r2 = s32_of(dx, dy, dz);
        const bool in = r2 < s.H2;
        if (COUNT) {
            a.n += (in && j != s.idx) ? 1 : 0;
        } else {
            float wt, gt;
            wendland_t(r2, s.invH, wt, gt);
            a.w.x += in ? wt : 0.f;
        }
    }
    __device__ __forceinline__ void pair2(const I& s, Acc& a, const float4& p0, const float4*, int,
                                          const float4& p1, const float4*, int) const {
        const float2 dx = make_float2(p0.x - s.x, p1.x - s.x), dy = make_float2(p0.y - s.y, p1.y - s.y),
                     dz = make_float2(p0.z - s.z, p1.z - s.z);
        const float2 r2 = s32_of2(dx, dy, dz);
        float2 wt, gt;
        wendland_t2(r2, s.invH, wt, gt);
        a.w = __fadd2_rn(a.w, f2sel(r2.x < s.H2, r2.y < s.H2, wt));
    }
    template <int GG>
    __device__ void reduce(Acc& a) const {
        if (COUNT) {
            a.n = slot_sum_i<GG>(a.n);
        } else {
            a.w.x = slot_sum<GG>(a.w.x + a.w.y);
        }
    }
    __device__ void finish(int k, const I& s, const Acc& a) const {
        if (COUNT) {
            cnt[gas_idx[k]] = a.n;
            return;
        }
        const float V = 1.f / (SIGMA_W * s.invH * s.invH * s.invH * a.w.x);
        gV[k] = V;
        gposV[k] = make_float4(s.x, s.y, s.z, V);
        if (Vout) Vout[gas_idx[k]] = V;
    }
};

// symmetric 3x3 / 3x3x3 index of the accumulated moments (CorPass accumulators)
__device__ __forceinline__ int sym2(int a, int b) {
    if (a > b) { int t = a; a = b; b = t; }
    return a == 0 ? b : (a == 1 ? 2 + b : 5);
}
__device__ __forceinline__ int sym3(int a, int b, int g) {
    int x = a, y = b, z = g, t;
    if (x > y) { t = x; x = y; y = t; }
    if (y > z) { t = y; y = z; z = t; }
    if (x > y) { t = x; x = y; y = t; }
    const int tab[3][3][3] = {{{0, 1, 2}, {0, 3, 4}, {0, 0, 5}},
                              {{0, 0, 0}, {0, 6, 7}, {0, 0, 8}},
                              {{0, 0, 0}, {0, 0, 0}, {0, 0, 9}}};
    return tab[x][y][z];
}

// O7 coefficients A, B, grad A, grad B of one particle from its accumulated moments (d = x_j - x_i
// convention, unscaled kernel: am* = sum V_j d.. wt, ag* = sum V_j d.. gt), 1/H its support
__device__ __forceinline__ void cor_coefficients(float invH, float am0, const float am1[3], const float am2[6],
                                                 const float ag0[3], const float ag1[6], const float ag2[10],
                                                 float& Ai, float Bi[3], float dAi[3], float dBi[3][3]) {
    const float c = SIGMA_W * invH * invH * invH;
    const float cg = c * invH * invH;
    // moments in x_ij = -d convention (O7), delta terms added here
    const float m0 = c * am0;
    float m1[3], m2[3][3], g0[3], g1[3][3], g2[3][3][3];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        m1[p] = -c * am1[p];
        g0[p] = -cg * ag0[p];
    }
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            m2[p][q] = c * am2[sym2(p, q)];
            g1[p][q] = cg * ag1[sym2(p, q)] + (p == q ? m0 : 0.f);
#pragma unroll
            for (int g = 0; g < 3; ++g)
                g2[p][q][g] = -cg * ag2[sym3(p, q, g)] + (p == g ? m1[q] : 0.f) + (q == g ? m1[p] : 0.f);
        }
    // fp32 cofactor inverse of m2
    const float c00 = m2[1][1] * m2[2][2] - m2[1][2] * m2[2][1];
    const float c01 = m2[1][2] * m2[2][0] - m2[1][0] * m2[2][2];
    const float c02 = m2[1][0] * m2[2][1] - m2[1][1] * m2[2][0];
    const float det = m2[0][0] * c00 + m2[0][1] * c01 + m2[0][2] * c02;
    const float tr = (m2[0][0] + m2[1][1] + m2[2][2]) * (1.f / 3.f);
    if (fabsf(det) < 1e-10f * tr * tr * tr) {
        Ai = 1.f / m0;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            Bi[p] = 0.f;
            dAi[p] = -g0[p] / (m0 * m0);
#pragma unroll
            for (int g = 0; g < 3; ++g) dBi[p][g] = 0.f;
        }
    } else {
        const float id = 1.f / det;
        float mi[3][3];
        mi[0][0] = c00 * id;
        mi[0][1] = (m2[0][2] * m2[2][1] - m2[0][1] * m2[2][2]) * id;
        mi[0][2] = (m2[0][1] * m2[1][2] - m2[0][2] * m2[1][1]) * id;
        mi[1][0] = c01 * id;
        mi[1][1] = (m2[0][0] * m2[2][2] - m2[0][2] * m2[2][0]) * id;
        mi[1][2] = (m2[0][2] * m2[1][0] - m2[0][0] * m2[1][2]) * id;
        mi[2][0] = c02 * id;
        mi[2][1] = (m2[0][1] * m2[2][0] - m2[0][0] * m2[2][1]) * id;
        mi[2][2] = (m2[0][0] * m2[1][1] - m2[0][1] * m2[1][0]) * id;
#pragma unroll
        for (int p = 0; p < 3; ++p) Bi[p] = -(mi[p][0] * m1[0] + mi[p][1] * m1[1] + mi[p][2] * m1[2]);
        Ai = 1.f / (m0 + Bi[0] * m1[0] + Bi[1] * m1[1] + Bi[2] * m1[2]);
#pragma unroll
        for (int g = 0; g < 3; ++g) {
            float rhs[3];
#pragma unroll
            for (int p = 0; p < 3; ++p)
                rhs[p] = g1[p][g] + g2[p][0][g] * Bi[0] + g2[p][1][g] * Bi[1] + g2[p][2][g] * Bi[2];
#pragma unroll
            for (int p = 0; p < 3; ++p) dBi[p][g] = -(mi[p][0] * rhs[0] + mi[p][1] * rhs[1] + mi[p][2] * rhs[2]);
        }
#pragma unroll
        for (int g = 0; g < 3; ++g) {
            float t = g0[g];
#pragma unroll
            for (int p = 0; p < 3; ++p) t += dBi[p][g] * m1[p] + Bi[p] * g1[p][g];
            dAi[g] = -Ai * Ai * t;
        }
    }
}

// ============================================================== a5 Corrections (upCor)
// Moments over gas j with s32 < H_i^2 (j incl. i), accumulated with d = x_j - x_i
// (x_ij = -d); the symmetric gradient moments need only 6 + 10 accumulators.
struct CorPass : HydCommon {
    static constexpr int PAY = 0;
    static constexpr bool SYM = false;
    static constexpr int UNROLL = 2;
    const float4* jrows;  // gposV (x, y, z, V)
    const float4* jpay;
    float* gcoef;  // 16 planes of n_gas
    int64_t ng;
    float *A, *B, *dA, *dB;  // caller planes (n)
    int64_t n;
    struct I { float x, y, z, H2, invH; };
    // moments, paired for packed FP32 (components named by their d indices):
    //   m1: (0, 1), 2;  m2: (00, 01), (02, 12), 11, 22;  likewise g0, g1;
    //   g2: (000, 001), (002, 012), (022, 122), 011, 111, 112, 222
    struct Acc {
        float m0, m1_2, g0_2, m2_11, m2_22, g1_11, g1_22, g2_011, g2_111, g2_112, g2_222;
        float2 m1_01, m2_a, m2_b, g0_01, g1_a, g1_b, g2_a, g2_b, g2_c;
    };
    __device__ void init(Acc& a) const {
        a.m0 = a.m1_2 = a.g0_2 = a.m2_11 = a.m2_22 = a.g1_11 = a.g1_22 = 0.f;
        a.g2_011 = a.g2_111 = a.g2_112 = a.g2_222 = 0.f;
        a.m1_01 = a.m2_a = a.m2_b = a.g0_01 = a.g1_a = a.g1_b = a.g2_a = a.g2_b = a.g2_c = make_float2(0.f, 0.f);
    }
    __device__ void load_i(int k, I& s) const { load_pos(gpos, k, s.x, s.y, s.z, s.H2, s.invH); }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I& s) const { return s.H2; }
    __device__ float jcut(const float4&) const { return 0.f; }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4*, int) const {
        const float2 d01 = __fadd2_rn(make_float2(jp.x, jp.y), make_float2(-s.x, -s.y));  // d = x_j - x_i
        const float d2 = jp.z - s.z;
        const float r2 = s32_of(d01.x, d01.y, d2);
        float wt, gt;
        wendland_t(r2, s.invH, wt, gt);
        const bool in = r2 < s.H2;
        const float2 wg = __fmul2_rn(make_float2(jp.w, jp.w), make_float2(wt, gt));
        const float w = in ? wg.x : 0.f;
        const float gw = in ? wg.y : 0.f;  // (times 1/H^2 in finish)
        const float2 wd01 = __fmul2_rn(make_float2(w, w), d01);
        const float wd2 = w * d2;
        a.m0 += w;
        a.m1_01 = __fadd2_rn(a.m1_01, wd01);
        a.m1_2 += wd2;
        a.m2_a = __ffma2_rn(make_float2(wd01.x, wd01.x), d01, a.m2_a);  // (00, 01)
        a.m2_b = __ffma2_rn(make_float2(wd2, wd2), d01, a.m2_b);        // (02, 12)
        a.m2_11 = fmaf(wd01.y, d01.y, a.m2_11);
        a.m2_22 = fmaf(wd2, d2, a.m2_22);
        const float2 gd01 = __fmul2_rn(make_float2(gw, gw), d01);
        const float gd2 = gw * d2;
        a.g0_01 = __fadd2_rn(a.g0_01, gd01);
        a.g0_2 += gd2;
        a.g1_a = __ffma2_rn(make_float2(gd01.x, gd01.x), d01, a.g1_a);
        a.g1_b = __ffma2_rn(make_float2(gd2, gd2), d01, a.g1_b);
        a.g1_11 = fmaf(gd01.y, d01.y, a.g1_11);
        a.g1_22 = fmaf(gd2, d2, a.g1_22);
        // fully symmetric third moment d_a d_b d_g gw
        const float2 e = __fmul2_rn(make_float2(gd01.x, gd01.x), d01);          // (e00, e01)
        a.g2_a = __ffma2_rn(make_float2(e.x, e.x), d01, a.g2_a);                // (000, 001)
        a.g2_b = __ffma2_rn(make_float2(d2, d2), e, a.g2_b);                    // (002, 012)
        a.g2_011 = fmaf(e.y, d01.y, a.g2_011);
        const float2 f = __fmul2_rn(gd01, make_float2(d2, d2));                 // (gd0 d2, gd1 d2)
        a.g2_c = __ffma2_rn(make_float2(d2, d2), f, a.g2_c);                    // (022, 122)
        const float e11 = gd01.y * d01.y;
        a.g2_111 = fmaf(e11, d01.y, a.g2_111);
        a.g2_112 = fmaf(e11, d2, a.g2_112);
        a.g2_222 = fmaf(gd2 * d2, d2, a.g2_222);
    }
    template <int GG>
    __device__ void reduce(Acc& a) const {
        float* p[11] = {&a.m0, &a.m1_2, &a.g0_2, &a.m2_11, &a.m2_22, &a.g1_11, &a.g1_22, &a.g2_011, &a.g2_111, &a.g2_112, &a.g2_222};
#pragma unroll
        for (int t = 0; t < 11; ++t) *p[t] = slot_sum<GG>(*p[t]);
        float2* q[9] = {&a.m1_01, &a.m2_a, &a.m2_b, &a.g0_01, &a.g1_a, &a.g1_b, &a.g2_a, &a.g2_b, &a.g2_c};
#pragma unroll
        for (int t = 0; t < 9; ++t) { q[t]->x = slot_sum<GG>(q[t]->x); q[t]->y = slot_sum<GG>(q[t]->y); }
    }
    __device__ static int s2(int a, int b) {  // symmetric 3x3 index
        if (a > b) { int t = a; a = b; b = t; }
        return a == 0 ? b : (a == 1 ? 2 + b : 5);
    }
    __device__ static int s3(int a, int b, int g) {  // symmetric 3x3x3 index
        int x = a, y = b, z = g, t;
        if (x > y) { t = x; x = y; y = t; }
        if (y > z) { t = y; y = z; z = t; }
        if (x > y) { t = x; x = y; y = t; }
        // sorted x <= y <= z
        const int tab[3][3][3] = {{{0, 1, 2}, {0, 3, 4}, {0, 0, 5}},
                                  {{0, 0, 0}, {0, 6, 7}, {0, 0, 8}},
                                  {{0, 0, 0}, {0, 0, 0}, {0, 0, 9}}};
        return tab[x][y][z];
    }
    __device__ void finish(int k, const I& s, const Acc& a) const {
        float Ai, Bi[3], dAi[3], dBi[3][3];
        // canonical index sets: m2 / g1 {00, 01, 02, 11, 12, 22}, g2 {000, 001, 002, 011, 012, 022, 111, 112, 122, 222}
        const float m1[3] = {a.m1_01.x, a.m1_01.y, a.m1_2};
        const float m2[6] = {a.m2_a.x, a.m2_a.y, a.m2_b.x, a.m2_11, a.m2_b.y, a.m2_22};
        const float g0[3] = {a.g0_01.x, a.g0_01.y, a.g0_2};
        const float g1[6] = {a.g1_a.x, a.g1_a.y, a.g1_b.x, a.g1_11, a.g1_b.y, a.g1_22};
        const float g2[10] = {a.g2_a.x, a.g2_a.y, a.g2_b.x, a.g2_011, a.g2_b.y, a.g2_c.x, a.g2_111, a.g2_112, a.g2_c.y,
                              a.g2_222};
        cor_coefficients(s.invH, a.m0, m1, m2, g0, g1, g2, Ai, Bi, dAi, dBi);
        float vals[16];
        vals[0] = Ai;
#pragma unroll
        for (int p = 0; p < 3; ++p) { vals[1 + p] = Bi[p]; vals[4 + p] = dAi[p]; }
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int g = 0; g < 3; ++g) vals[7 + 3 * p + g] = dBi[p][g];
#pragma unroll
        for (int t = 0; t < 16; ++t) gcoef[(int64_t)t * ng + k] = vals[t];
        const int64_t i = gas_idx[k];
        if (A) A[i] = Ai;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            if (B) B[p * n + i] = Bi[p];
            if (dA) dA[p * n + i] = dAi[p];
        }
        if (dB)
#pragma unroll
            for (int t = 0; t < 9; ++t) dB[t * n + i] = vals[7 + t];
    }
};

// ---------------------------------------------------------------- accel records
// The accel/du-dt pass reads a neighbour's state as one 9-float4 record (ExtPass::finish writes it),
// laid out so that the packed-FP32 pair terms (AccPass::pair) find their operand pairs aligned in
// the registers of 128-bit loads: (g = 0, 1) pairs of B, dA, dB for the corrected kernel
// gradient, (p = 0, 1) pairs of grad v for the limiter, and (x, y) of v.
//   0: dB0 dB1 dB3 dB4 | 1: dB6 dB7 B0 B1 | 2: dAh0 dAh1 dv0 dv3 | 3: dv1 dv4 dv2 dv5
//   4: v0 v1 dB2 dB5   | 5: dB8 B2 dAh2 Ah | 6: dv6 dv7 dv8 v2     | 7: V P rho cs
//   8: 1/H H^2 m u (the particle's own use only)
// dB[3p + g] = d B_g / d x_p, dv[3a + b] = d v^a / d x_b, Ah = sigma A / H^3, dAh = sigma grad A / H^3.
// (The 9-float4 stride is odd, so staged records of consecutive slots start in different
// shared-memory bank groups; an 8-float4 stride put every slot's component in the same group.)
__device__ __forceinline__ void write_rec(float4* rec, float Ah, const float B[3], const float dAh[3], const float dB[9],
                                          float vx, float vy, float vz, const float dv[9], float V, float P, float rho,
                                          float cs, float invH, float H2, float m, float u) {
    rec[0] = make_float4(dB[0], dB[1], dB[3], dB[4]);
    rec[1] = make_float4(dB[6], dB[7], B[0], B[1]);
    rec[2] = make_float4(dAh[0], dAh[1], dv[0], dv[3]);
    rec[3] = make_float4(dv[1], dv[4], dv[2], dv[5]);
    rec[4] = make_float4(vx, vy, dB[2], dB[5]);
    rec[5] = make_float4(dB[8], B[2], dAh[2], Ah);
    rec[6] = make_float4(dv[6], dv[7], dv[8], vz);
    rec[7] = make_float4(V, P, rho, cs);
    rec[8] = make_float4(invH, H2, m, u);
}

// ============================================================== a6 Extras (upBarEx)
// rho = sum m_j W^R_ij, P = (gamma-1) rho u, c = sqrt(gamma P / rho),
// d_b v^a = sum V_j (v^a_j - v^a_i) d_b W^R_ij ; the epilogue also packs the accel
// record (9 float4) of particle i for a7/a8.
struct ExtPass : HydCommon {
    static constexpr int PAY = 1;
    static constexpr bool SYM = false;
    static constexpr int UNROLL = 2;
    const float4* jrows;  // gposV (x, y, z, V)
    const float4* jpay;   // gvel (vx, vy, vz, m)
    const float* gV;
    const float* gcoef;
    const float4* gvel;  // (vx, vy, vz, m)
    const float* gu;
    float4* grec;
    int64_t ng, n;
    float gamma;
    float *rho, *P, *cs, *dv;  // caller
    struct I {
        float x, y, z, H2, invH;
        float A, B[3], dA[3], dB[9];
        float vx, vy, vz;
    };
    // grad v sums g[3a + b] (a: velocity component, b: derivative) paired over b = 0, 1:
    // g01[a] = (g[3a], g[3a + 1]), g2[a] = g[3a + 2]
    struct Acc { float rho, g2[3]; float2 g01[3]; };
    __device__ void init(Acc& a) const {
        a.rho = 0.f;
#pragma unroll
        for (int t = 0; t < 3; ++t) { a.g2[t] = 0.f; a.g01[t] = make_float2(0.f, 0.f); }
    }
    __device__ void load_i(int k, I& s) const {
        load_pos(gpos, k, s.x, s.y, s.z, s.H2, s.invH);
        s.A = gcoef[k];
#pragma unroll
        for (int p = 0; p < 3; ++p) { s.B[p] = gcoef[(1 + p) * ng + k]; s.dA[p] = gcoef[(4 + p) * ng + k]; }
#pragma unroll
        for (int t = 0; t < 9; ++t) s.dB[t] = gcoef[(7 + t) * ng + k];
        const float4 v = gvel[k];
        s.vx = v.x; s.vy = v.y; s.vz = v.z;
    }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I& s) const { return s.H2; }
    __device__ float jcut(const float4&) const { return 0.f; }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4* pay, int) const {
        // x_ij = x_i - x_j
        const float2 x01 = __fadd2_rn(make_float2(s.x, s.y), make_float2(-jp.x, -jp.y));
        const float x2 = s.z - jp.z;
        const float r2 = s32_of(x01.x, x01.y, x2);
        const bool in = r2 < s.H2;  // branch-free: out-of-range pairs add exact zeros
        float wt, gt;
        wendland_t(r2, s.invH, wt, gt);
        wt = in ? wt : 0.f;
        gt = in ? gt * (s.invH * s.invH) : 0.f;
        const float lin = fmaf(s.B[2], x2, fmaf(s.B[1], x01.y, fmaf(s.B[0], x01.x, 1.f)));
        const float4 vj = pay[0];
        a.rho = fmaf(vj.w, s.A * lin * wt, a.rho);
        const float alg = s.A * lin * gt;
        // t1_g = sum_p dB[3p + g] x_p + B_g, packed over g = 0, 1
        const float2 t01 = __ffma2_rn(make_float2(s.dB[6], s.dB[7]), make_float2(x2, x2),
                                      __ffma2_rn(make_float2(s.dB[3], s.dB[4]), make_float2(x01.y, x01.y),
                                                 __ffma2_rn(make_float2(s.dB[0], s.dB[1]), make_float2(x01.x, x01.x),
                                                            make_float2(s.B[0], s.B[1]))));
        const float t2 = fmaf(s.dB[8], x2, fmaf(s.dB[5], x01.y, fmaf(s.dB[2], x01.x, s.B[2])));
        // gw_g = wt (dA_g lin + A t1_g) + alg x_g
        const float2 gw01 = __ffma2_rn(make_float2(alg, alg), x01,
                                       __fmul2_rn(make_float2(wt, wt),
                                                  __ffma2_rn(make_float2(s.dA[0], s.dA[1]), make_float2(lin, lin),
                                                             __fmul2_rn(make_float2(s.A, s.A), t01))));
        const float gw2 = fmaf(alg, x2, wt * fmaf(s.dA[2], lin, s.A * t2));
        const float Vj = jp.w;
        const float2 e01 = __fmul2_rn(make_float2(Vj, Vj), __fadd2_rn(make_float2(vj.x, vj.y), make_float2(-s.vx, -s.vy)));
        const float e[3] = {e01.x, e01.y, Vj * (vj.z - s.vz)};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            a.g01[c] = __ffma2_rn(make_float2(e[c], e[c]), gw01, a.g01[c]);
            a.g2[c] = fmaf(e[c], gw2, a.g2[c]);
        }
    }
    template <int GG>
    __device__ void reduce(Acc& a) const {
        a.rho = slot_sum<GG>(a.rho);
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            a.g2[t] = slot_sum<GG>(a.g2[t]);
            a.g01[t].x = slot_sum<GG>(a.g01[t].x);
            a.g01[t].y = slot_sum<GG>(a.g01[t].y);
        }
    }
    __device__ void finish(int k, const I& s, const Acc& a) const {
        const float c = SIGMA_W * s.invH * s.invH * s.invH;
        const float r = c * a.rho;
        const float u = gu[k];
        const float Pk = (gamma - 1.f) * r * u;
        const float ck = sqrtf(gamma * Pk / r);
        float g[9];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            g[3 * t] = c * a.g01[t].x;
            g[3 * t + 1] = c * a.g01[t].y;
            g[3 * t + 2] = c * a.g2[t];
        }
        const float V = gV[k];
        const float4 vm = gvel[k];
        const float dAh[3] = {c * s.dA[0], c * s.dA[1], c * s.dA[2]};
        write_rec(grec + (int64_t)k * 9, c * s.A, s.B, dAh, s.dB, vm.x, vm.y, vm.z, g, V, Pk, r, ck, s.invH, s.H2, vm.w, u);
        const int64_t i = gas_idx[k];
        if (rho) rho[i] = r;
        if (P) P[i] = Pk;
        if (cs) cs[i] = ck;
        if (dv)
#pragma unroll
            for (int t = 0; t < 9; ++t) dv[t * n + i] = g[t];
    }
};

// ============================================================== a5 + a6 in ONE list walk
// Corrections and Extras from one walk of each gas particle's list: Extras' sums are linear in
// quantities known per pair, so with x = x_ij = -d, W~ = wt, G~ = gt (unscaled) and e = V_j (v_j - v_i)
//   rho / c      = A (M0 + B.M1x),                       M0 = sum m_j W~,  M1x_c = sum m_j W~ x_c
//   d_b v^a / c  = dA_b (S0_a + B.S1x_a) + A (sum_c dB_c,b S1x_ac + B_b S0_a)
//                + (1/H^2) A (T0x_ab + sum_c B_c T1x_abc)
//   S0_a = sum e_a W~, S1x_ac = sum e_a W~ x_c, T0x_ab = sum e_a G~ x_b, T1x_abc = sum e_a G~ x_b x_c
// (c = sigma/H^3): the same sums as ExtPass's per-pair corrected-kernel gradient (O7, O8), reordered
// — accumulated during the Corrections walk, combined with i's coefficients in the epilogue, so the
// second walk (and its kernel evaluations) is gone.  43 accumulators on top of Corrections' 29.
struct CorExtPass : HydCommon {
    static constexpr int PAY = 1;
    static constexpr bool SYM = false;
    static constexpr int UNROLL = 1;
    const float4* jrows;  // gposV (x, y, z, V)
    const float4* jpay;   // gvel (vx, vy, vz, m)
    const float* gV;
    const float4* gvel;
    const float* gu;
    float4* grec;
    int64_t ng, n;
    float gamma;
    float *A, *B, *dA, *dB, *rho, *P, *cs, *dv;  // caller (may be null)
    struct I { float x, y, z, H2, invH, vx, vy, vz; };
    struct Acc {
        float m0, m1[3], m2[6], g0[3], g1[6], g2[10];  // Corrections (d convention)
        float M0, M1[3], S0[3], S1[9], T0[9], T1[18];   // Extras moments (d convention)
    };
    __device__ void init(Acc& a) const {
        a.m0 = a.M0 = 0.f;
#pragma unroll
        for (int t = 0; t < 3; ++t) a.m1[t] = a.g0[t] = a.M1[t] = a.S0[t] = 0.f;
#pragma unroll
        for (int t = 0; t < 6; ++t) a.m2[t] = a.g1[t] = 0.f;
#pragma unroll
        for (int t = 0; t < 10; ++t) a.g2[t] = 0.f;
#pragma unroll
        for (int t = 0; t < 9; ++t) a.S1[t] = a.T0[t] = 0.f;
#pragma unroll
        for (int t = 0; t < 18; ++t) a.T1[t] = 0.f;
    }
    __device__ void load_i(int k, I& s) const {
        load_pos(gpos, k, s.x, s.y, s.z, s.H2, s.invH);
        const float4 v = gvel[k];
        s.vx = v.x; s.vy = v.y; s.vz = v.z;
    }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I& s) const { return s.H2; }
    __device__ float jcut(const float4&) const { return 0.f; }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4* pay, int) const {
        const float d0 = jp.x - s.x, d1 = jp.y - s.y, d2 = jp.z - s.z;  // d = x_j - x_i, exact (O1)
        const float r2 = s32_of(d0, d1, d2);
        float wt, gt;
        wendland_t(r2, s.invH, wt, gt);
        const bool in = r2 < s.H2;
        wt = in ? wt : 0.f;
        gt = in ? gt : 0.f;
        const float dd[6] = {d0 * d0, d0 * d1, d0 * d2, d1 * d1, d1 * d2, d2 * d2};
        const float d[3] = {d0, d1, d2};
        // Corrections' moments
        const float w = jp.w * wt, gw = jp.w * gt;
        a.m0 += w;
#pragma unroll
        for (int t = 0; t < 3; ++t) { a.m1[t] = fmaf(w, d[t], a.m1[t]); a.g0[t] = fmaf(gw, d[t], a.g0[t]); }
#pragma unroll
        for (int t = 0; t < 6; ++t) { a.m2[t] = fmaf(w, dd[t], a.m2[t]); a.g1[t] = fmaf(gw, dd[t], a.g1[t]); }
        const float gd0 = gw * d0, gd1 = gw * d1, gd2 = gw * d2;
        // symmetric third moment, index set 000,001,002,011,012,022,111,112,122,222
        a.g2[0] = fmaf(gd0, dd[0], a.g2[0]);
        a.g2[1] = fmaf(gd0, dd[1], a.g2[1]);
        a.g2[2] = fmaf(gd0, dd[2], a.g2[2]);
        a.g2[3] = fmaf(gd0, dd[3], a.g2[3]);
        a.g2[4] = fmaf(gd0, dd[4], a.g2[4]);
        a.g2[5] = fmaf(gd0, dd[5], a.g2[5]);
        a.g2[6] = fmaf(gd1, dd[3], a.g2[6]);
        a.g2[7] = fmaf(gd1, dd[4], a.g2[7]);
        a.g2[8] = fmaf(gd1, dd[5], a.g2[8]);
        a.g2[9] = fmaf(gd2, dd[5], a.g2[9]);
        // Extras' moments
        const float4 vj = pay[0];
        const float mW = vj.w * wt;
        a.M0 += mW;
#pragma unroll
        for (int t = 0; t < 3; ++t) a.M1[t] = fmaf(mW, d[t], a.M1[t]);
        const float e[3] = {jp.w * (vj.x - s.vx), jp.w * (vj.y - s.vy), jp.w * (vj.z - s.vz)};
#pragma unroll
        for (int al = 0; al < 3; ++al) {
            const float eW = e[al] * wt, eG = e[al] * gt;
            a.S0[al] += eW;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                a.S1[3 * al + t] = fmaf(eW, d[t], a.S1[3 * al + t]);
                a.T0[3 * al + t] = fmaf(eG, d[t], a.T0[3 * al + t]);
            }
#pragma unroll
            for (int t = 0; t < 6; ++t) a.T1[6 * al + t] = fmaf(eG, dd[t], a.T1[6 * al + t]);
        }
    }
    template <int GG>
    __device__ void reduce(Acc& a) const {
        float* v = reinterpret_cast<float*>(&a);
#pragma unroll
        for (int t = 0; t < (int)(sizeof(Acc) / sizeof(float)); ++t) v[t] = slot_sum<GG>(v[t]);
    }
    __device__ void finish(int k, const I& s, const Acc& a) const {
        float Ai, Bi[3], dAi[3], dBi[3][3];
        cor_coefficients(s.invH, a.m0, a.m1, a.m2, a.g0, a.g1, a.g2, Ai, Bi, dAi, dBi);
        const float c = SIGMA_W * s.invH * s.invH * s.invH;
        const float cg = c * s.invH * s.invH;
        // x = -d: M1x = -M1, S1x = -S1, T0x = -T0, T1x = T1
        const float r = c * Ai * (a.M0 - (Bi[0] * a.M1[0] + Bi[1] * a.M1[1] + Bi[2] * a.M1[2]));
        float g[9];
#pragma unroll
        for (int al = 0; al < 3; ++al) {
            const float* S1 = a.S1 + 3 * al;
            const float* T0 = a.T0 + 3 * al;
            const float* T1 = a.T1 + 6 * al;
            const float lin = a.S0[al] - (Bi[0] * S1[0] + Bi[1] * S1[1] + Bi[2] * S1[2]);
#pragma unroll
            for (int be = 0; be < 3; ++be) {
                const float t1 = -(dBi[0][be] * S1[0] + dBi[1][be] * S1[1] + dBi[2][be] * S1[2]) + Bi[be] * a.S0[al];
                float t3 = -T0[be];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) t3 += Bi[cc] * T1[sym2(be, cc)];
                g[3 * al + be] = c * (dAi[be] * lin + Ai * t1) + cg * Ai * t3;
            }
        }
        const float u = gu[k];
        const float Pk = (gamma - 1.f) * r * u;
        const float ck = sqrtf(gamma * Pk / r);
        const float V = gV[k];
        const float4 vm = gvel[k];
        const float dAh[3] = {c * dAi[0], c * dAi[1], c * dAi[2]};
        const float dBf[9] = {dBi[0][0], dBi[0][1], dBi[0][2], dBi[1][0], dBi[1][1], dBi[1][2], dBi[2][0], dBi[2][1], dBi[2][2]};
        write_rec(grec + (int64_t)k * 9, c * Ai, Bi, dAh, dBf, vm.x, vm.y, vm.z, g, V, Pk, r, ck, s.invH, s.H2, vm.w, u);
        const int64_t i = gas_idx[k];
        if (A) A[i] = Ai;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            if (B) B[p * n + i] = Bi[p];
            if (dA) dA[p * n + i] = dAi[p];
        }
        if (dB)
#pragma unroll
            for (int t = 0; t < 9; ++t) dB[t * n + i] = dBi[t / 3][t % 3];
        if (rho) rho[i] = r;
        if (P) P[i] = Pk;
        if (cs) cs[i] = ck;
        if (dv)
#pragma unroll
            for (int t = 0; t < 9; ++t) dv[t * n + i] = g[t];
    }
};

// ============================================================== a7 + a8 Acceleration, Energy
// Antisymmetrised CRK-SPH (O9): G_ij = (grad W^R_ij - grad W^R_ji)/2, each half with its
// own particle's coefficients and H; artificial viscosity with a van Leer limited
// midpoint velocity reconstruction.  Symmetric predicate s32 < max(H_i^2, H_j^2).
// ============================================================== count mode of the list walks
// Integer payload: the pairs a gas pass evaluates while it walks
// the neighbour lists (or culls on the fly for flagged rows), j != i: the gather predicate
// s32 < H_i^2 of corrections/extras (SYMP false) or the symmetric s32 < max(H_i^2, H_j^2) of
// accel/du-dt (SYMP true).  Positions are staged from gpos (x, y, z, H): the same slots.
template <bool SYMP>
struct ListCountPass : HydCommon {
    static constexpr int PAY = 0;
    static constexpr bool SYM = SYMP;
    static constexpr int UNROLL = 4;
    const float4* jrows;  // gpos
    const float4* jpay;
    int32_t* cnt;
    struct I { float x, y, z, H2, invH; int idx; };
    struct Acc { int n; };
    __device__ void init(Acc& a) const { a.n = 0; }
    __device__ void load_i(int k, I& s) const { load_pos(gpos, k, s.x, s.y, s.z, s.H2, s.invH); s.idx = k; }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I& s) const { return s.H2; }
    __device__ float jcut(const float4& jp) const { return __fmul_rn(jp.w, jp.w); }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4*, int j) const {
        const float r2 = s32_of(jp.x - s.x, jp.y - s.y, jp.z - s.z);
        const bool in = SYMP ? r2 < fmaxf(s.H2, __fmul_rn(jp.w, jp.w)) : r2 < s.H2;
        a.n += (in && j != s.idx) ? 1 : 0;
    }
    template <int GG>
    __device__ void reduce(Acc& a) const { a.n = slot_sum_i<GG>(a.n); }
    __device__ void finish(int k, const I&, const Acc& a) const { cnt[gas_idx[k]] = a.n; }
};

// ============================================================== a7 + a8 pair terms, packed FP32
// The antisymmetrised pair terms of one pair (i, j) from the two accel records (write_rec layout),
// x_ij = x01, x2 (x_i - x_j), r2 = s32: the corrected kernel gradients of both particles (the
// kernel factors of i and j packed, the gradients packed over components), the limiter and the
// artificial viscosity.  Returns G_ij = (grad W^R_ij - grad W^R_ji) / 2, PQ = P_i + P_j + Q_ij,
// Qh = Q_ij / 2 and vG = v_ij . G_ij; the i-centric pass makes m_i dv_i/dt += -V_i V_j PQ G and
// m_i du_i/dt += V_i V_j (P_i + Qh) vG from them, the Newton-3 pass both particles' terms.
struct AccTerms {
    float2 G01;
    float G2, PQ, Qh, vG;
};
__device__ __forceinline__ static void grad_wr2(const float4* Q, float sg, float2 x01, float x2, float wt, float gt,
                                               float lin, float2& o01, float& o2) {
    const float2 dB01 = make_float2(Q[0].x, Q[0].y), dB34 = make_float2(Q[0].z, Q[0].w);
    const float2 dB67 = make_float2(Q[1].x, Q[1].y), B01 = make_float2(Q[1].z, Q[1].w);
    const float2 dAh01 = make_float2(Q[2].x, Q[2].y);
    const float dB2 = Q[4].z, dB5 = Q[4].w, dB8 = Q[5].x, B2 = Q[5].y, dAh2 = Q[5].z, Ah = Q[5].w;
    const float sx0 = sg * x01.x, sx1 = sg * x01.y, sx2 = sg * x2;
    // t1_g = sg sum_p dB[3p + g] x_p + B_g
    const float2 t01 = __ffma2_rn(dB67, make_float2(sx2, sx2), __ffma2_rn(dB34, make_float2(sx1, sx1),
                                                                         __ffma2_rn(dB01, make_float2(sx0, sx0), B01)));
    const float t2 = fmaf(dB8, sx2, fmaf(dB5, sx1, fmaf(dB2, sx0, B2)));
    const float alg = Ah * lin * gt * sg;
    // out_g = wt (dAh_g lin + Ah t1_g) + alg sg x_g
    o01 = __ffma2_rn(make_float2(alg, alg), x01,
                     __fmul2_rn(make_float2(wt, wt), __ffma2_rn(dAh01, make_float2(lin, lin), __fmul2_rn(make_float2(Ah, Ah), t01))));
    o2 = fmaf(alg, x2, wt * fmaf(dAh2, lin, Ah * t2));
}
__device__ __forceinline__ AccTerms acc_terms(const float4* Ri, const float4* Q, float Hj, float2 x01, float x2, float r2,
                                              float Cl, float Cq, float e2) {
    const float r = sqrtf(r2);
    // Wendland C4 factors of i (.x, support H_i) and j (.y, H_j), packed
    const float2 ih = make_float2(Ri[8].x, 1.f / Hj);
    const float2 q = __fmul2_rn(make_float2(r, r), ih);
    float2 t = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-q.x, -q.y));
    t = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
    const float2 t2 = __fmul2_rn(t, t);
    const float2 t5 = __fmul2_rn(__fmul2_rn(t2, t2), t);
    const float2 wt = __fmul2_rn(__fmul2_rn(t5, t),
                                 __ffma2_rn(q, __ffma2_rn(q, make_float2(35.f / 3.f, 35.f / 3.f), make_float2(6.f, 6.f)),
                                            make_float2(1.f, 1.f)));
    const float2 ih2 = __fmul2_rn(ih, ih);
    const float2 gt = __fmul2_rn(__fmul2_rn(make_float2(-56.f / 3.f, -56.f / 3.f), ih2),
                                 __fmul2_rn(t5, __ffma2_rn(make_float2(5.f, 5.f), q, make_float2(1.f, 1.f))));
    // lin = 1 + B_i.x_ij (i), 1 - B_j.x_ij (j)
    const float lin_i = fmaf(Ri[5].y, x2, fmaf(Ri[1].w, x01.y, fmaf(Ri[1].z, x01.x, 1.f)));
    const float lin_j = fmaf(-Q[5].y, x2, fmaf(-Q[1].w, x01.y, fmaf(-Q[1].z, x01.x, 1.f)));
    float2 gi01, gj01;
    float gi2, gj2;
    grad_wr2(Ri, 1.f, x01, x2, wt.x, gt.x, lin_i, gi01, gi2);
    grad_wr2(Q, -1.f, x01, x2, wt.y, gt.y, lin_j, gj01, gj2);
    AccTerms T;
    T.G01 = __fmul2_rn(make_float2(0.5f, 0.5f), __fadd2_rn(gi01, make_float2(-gj01.x, -gj01.y)));
    T.G2 = 0.5f * (gi2 - gj2);
    // limiter on x.grad v.x: gv_p = sum_b dv[3p + b] x_b, packed over p = 0, 1
    const float2 gvi01 = __ffma2_rn(make_float2(Ri[3].z, Ri[3].w), make_float2(x2, x2),
                                    __ffma2_rn(make_float2(Ri[3].x, Ri[3].y), make_float2(x01.y, x01.y),
                                               __fmul2_rn(make_float2(Ri[2].z, Ri[2].w), make_float2(x01.x, x01.x))));
    const float2 gvj01 = __ffma2_rn(make_float2(Q[3].z, Q[3].w), make_float2(x2, x2),
                                    __ffma2_rn(make_float2(Q[3].x, Q[3].y), make_float2(x01.y, x01.y),
                                               __fmul2_rn(make_float2(Q[2].z, Q[2].w), make_float2(x01.x, x01.x))));
    const float gvi2 = fmaf(Ri[6].z, x2, fmaf(Ri[6].y, x01.y, Ri[6].x * x01.x));
    const float gvj2 = fmaf(Q[6].z, x2, fmaf(Q[6].y, x01.y, Q[6].x * x01.x));
    const float2 xi = __fmul2_rn(x01, gvi01), xj = __fmul2_rn(x01, gvj01);
    const float xgi = fmaf(x2, gvi2, xi.x + xi.y);
    const float xgj = fmaf(x2, gvj2, xj.x + xj.y);
    // phi = 4r/(1+r)^2 with r = xgi/xgj, written as 4 xgi xgj / (xgi + xgj)^2 (r > 0 <=> xgi xgj > 0)
    const float pr = xgi * xgj;
    const float sm = xgi + xgj;
    const float phi = pr > 0.f ? fminf(1.f, 4.f * pr / (sm * sm)) : 0.f;
    const float hp = -0.5f * phi;
    const float2 vij01 = __fadd2_rn(make_float2(Ri[4].x, Ri[4].y), make_float2(-Q[4].x, -Q[4].y));
    const float vij2 = Ri[6].w - Q[6].w;
    const float2 vs01 = __ffma2_rn(make_float2(hp, hp), __fadd2_rn(gvi01, gvj01), vij01);
    const float vs2 = fmaf(hp, gvi2 + gvj2, vij2);
    const float2 vx = __fmul2_rn(vs01, x01);
    const float vsx = fmaf(vs2, x2, vx.x + vx.y);
    // mu_i, mu_j packed: min(0, vsx / H / (r^2 / H^2 + eps^2))
    const float2 den = __ffma2_rn(make_float2(r2, r2), ih2, make_float2(e2, e2));
    const float2 mu = make_float2(fminf(0.f, vsx * ih.x / den.x), fminf(0.f, vsx * ih.y / den.y));
    const float Qv = Ri[7].z * mu.x * (Cq * mu.x - Cl * Ri[7].w) + Q[7].z * mu.y * (Cq * mu.y - Cl * Q[7].w);
    T.PQ = Ri[7].y + Q[7].y + Qv;
    T.Qh = 0.5f * Qv;
    const float2 vg = __fmul2_rn(vij01, T.G01);
    T.vG = fmaf(vij2, T.G2, vg.x + vg.y);
    return T;
}

template <bool COUNT, int BATCH_ = 32>
struct AccPass : HydCommon {
    static constexpr int PAY = COUNT ? 0 : 9;
    static constexpr bool SYM = true;
    static constexpr int UNROLL = 1;
    static constexpr int BATCH = COUNT ? 0 : BATCH_;
    static constexpr bool IREC = !COUNT;  // list walks stage the i-records (pairs.cuh)
    const float4* jrows;  // gpos (x, y, z, H)
    const float4* jpay;   // grec
    const float4* grec;
    float Cl, Cq, e2, dt;
    int64_t n, ng;
    float *ahx, *ahy, *ahz, *dudt, *vx, *vy, *vz, *u;
    int32_t* cnt;
    struct I { float x, y, z; int idx; float4 R[9]; };  // position and own record (write_rec layout)
    struct Acc { float2 a01; float a2, du; int nn; };
    __device__ void init(Acc& a) const { a.a01 = make_float2(0.f, 0.f); a.a2 = a.du = 0.f; a.nn = 0; }
    __device__ void load_i(int k, I& s) const {
        const float4 p = gpos[k];
        s.x = p.x; s.y = p.y; s.z = p.z; s.idx = k;
        if (COUNT) { s.R[8].y = __fmul_rn(p.w, p.w); return; }
#pragma unroll
        for (int t = 0; t < 9; ++t) s.R[t] = grec[9 * (int64_t)k + t];
    }
    __device__ void load_i_staged(int k, const float4& p, const float4* rec9, I& s) const {
        s.x = p.x; s.y = p.y; s.z = p.z; s.idx = k;
#pragma unroll
        for (int t = 0; t < 9; ++t) s.R[t] = rec9[t];
    }
    __device__ float ix(const I& s) const { return s.x; }
    __device__ float iy(const I& s) const { return s.y; }
    __device__ float iz(const I& s) const { return s.z; }
    __device__ float cut(const I& s) const { return s.R[8].y; }
    __device__ float jcut(const float4& jp) const { return __fmul_rn(jp.w, jp.w); }
    __device__ __forceinline__ bool in(const I& s, const float4& jp) const {
        return s32_of(s.x - jp.x, s.y - jp.y, s.z - jp.z) < fmaxf(s.R[8].y, __fmul_rn(jp.w, jp.w));
    }
    __device__ __forceinline__ void pair(const I& s, Acc& acc, const float4& jp, const float4* pay, int j) const {
        const float2 x01 = __fadd2_rn(make_float2(s.x, s.y), make_float2(-jp.x, -jp.y));  // x_ij, exact (O1)
        const float x2 = s.z - jp.z;
        const float r2 = s32_of(x01.x, x01.y, x2);
        const bool in = r2 < fmaxf(s.R[8].y, __fmul_rn(jp.w, jp.w));
        if (COUNT) {
            acc.nn += (in && j != s.idx) ? 1 : 0;
            return;
        }
        if (!in) return;
        float4 Q[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) Q[t] = pay[t];
        const AccTerms T = acc_terms(s.R, Q, jp.w, x01, x2, r2, Cl, Cq, e2);
        const float fa = -Q[7].x * T.PQ;                       // -V_j (P_i + P_j + Q)
        const float fu = Q[7].x * (s.R[7].y + T.Qh) * T.vG;   // V_j (P_i + Q/2) v_ij.G
        acc.a01 = __ffma2_rn(make_float2(fa, fa), T.G01, acc.a01);
        acc.a2 = fmaf(fa, T.G2, acc.a2);
        acc.du += fu;
    }
    template <int GG>
    __device__ void reduce(Acc& a) const {
        if (COUNT) {
            a.nn = slot_sum_i<GG>(a.nn);
            return;
        }
        a.a01.x = slot_sum<GG>(a.a01.x);
        a.a01.y = slot_sum<GG>(a.a01.y);
        a.a2 = slot_sum<GG>(a.a2);
        a.du = slot_sum<GG>(a.du);
    }
    __device__ void finish(int k, const I& s, const Acc& a) const {
        const int64_t i = gas_idx[k];
        if (COUNT) {
            cnt[i] = a.nn;
            return;
        }
        const float f = s.R[7].x / s.R[8].z;  // V / m
        const float a0 = f * a.a01.x, a1 = f * a.a01.y, a2 = f * a.a2, du = f * a.du;
        if (ahx) { ahx[i] = a0; ahy[i] = a1; ahz[i] = a2; }
        if (dudt) dudt[i] = du;
        if (dt != 0.f) {
            vx[i] = fmaf(dt, a0, vx[i]);
            vy[i] = fmaf(dt, a1, vy[i]);
            vz[i] = fmaf(dt, a2, vz[i]);
            u[i] = fmaf(dt, du, u[i]);
        }
    }
};

// ============================================================== a7 + a8, Newton-3 over the lists
// Each unordered pair {i, j} is evaluated once, in the row of its lower gas rank (i's list holds
// every j with s32 < max(H_i^2, H_j^2), a symmetric predicate, so j's list holds i): one CTA per
// gas i-leaf row, the row's j-records staged by TMA in rounds of ENT entries with its i-records
// and i-lists (16-bit staging slots, copied to shared memory so that skipping the entries with a
// lower rank is a shared-memory scan, not a chain of global loads).  The pair terms are the
// packed ones of the i-centric pass (acc_terms); i's sums stay in registers (4 lanes per i), j's
// terms go to a float4 (a, du/dt) accumulator with red.global.add.v4.f32.  Only when no row is
// flagged (every list complete) and the domain is whole (a ghost has no row of its own);
// otherwise the CTAs exit and the gated i-centric kernels run.
struct AccSymListArgs {
    const float4* gpos;  // (x, y, z, H)
    const float4* grec;  // accel records
    RowView rv;
    ListView lv;
    float4* acc;         // (a, du/dt) sums, zeroed
    int64_t ng;
    float Cl, Cq, e2;
};

constexpr int ASL_NW = 8, ASL_G = 8, ASL_ENT = 64;
using AslSmem = ListSmem<9, ASL_ENT, true>;
constexpr int ASL_LIST_OFF = (int)((sizeof(AslSmem) + 127) / 128 * 128);  // the row's lists follow

__global__ void __launch_bounds__(ASL_NW * 32, 2) acc_symlist_kernel(const AccSymListArgs A) {
    constexpr int S = 32 / ASL_G;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AslSmem& sm = *reinterpret_cast<AslSmem*>(smem_raw);
    uint16_t* lst = reinterpret_cast<uint16_t*>(smem_raw + ASL_LIST_OFF);
    const RowView& rv = A.rv;
    const ListView& lv = A.lv;
    if (*lv.nfrows != 0 || !row_selected(rv, blockIdx.x)) return;
    const int a = blockIdx.x;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int il = lane / S, sl = lane % S;
    const int ibase = warp * ASL_G;
    const int cap = lv.cap;
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar, 1);
        mbar_fence_init();
    }
    uint32_t phase = 0;
    const int ifirst = rv.ifirst[a], icount = rv.icount[a];
    const bool wactive = ibase < icount;
    const bool ivalid = ibase + il < icount;
    const int ki = ifirst + ibase + (ivalid ? il : 0);
    const int rbeg = rv.row_off[a], rend = rv.row_end[a];
    IStage ist;
    ist.grec = A.grec; ist.gpos = A.gpos; ist.ncnt = lv.ncnt;
    ist.ifirst = ifirst; ist.icount = icount;
    // the row's lists (consecutive gas ranks: one contiguous block; cap is a multiple of 8)
    ist.lsrc = lv.nbr + (int64_t)ifirst * cap;
    ist.ldst = lst;
    ist.lbytes = (uint32_t)(icount * cap * (int)sizeof(uint16_t));
    const uint16_t* L = lst + (ibase + il) * cap;
    float4 Ri[9];
    float ix = 0.f, iy = 0.f, iz = 0.f;
    int nl = 0, lp = sl, tn = 0x7fffffff;
    float2 s01 = make_float2(0.f, 0.f);
    float s2 = 0.f, s3 = 0.f;
    for (int e0 = rbeg; e0 < rend; e0 += ASL_ENT) {
        const int nent = min(ASL_ENT, rend - e0);
        stage_list_round<9, ASL_NW, ASL_ENT, true>(sm, rv, A.gpos, A.grec, e0, nent, phase,
                                                   e0 == rbeg ? &ist : nullptr);
        if (e0 == rbeg && wactive) {  // i-data from the staged copy
            const int ii = ki - ifirst;
            const float4 p = sm.ipos[ii];
            ix = p.x; iy = p.y; iz = p.z;
#pragma unroll
            for (int t = 0; t < 9; ++t) Ri[t] = sm.irec[ii * 9 + t];
            nl = ivalid ? sm.icnt[ii + (ifirst & 3)] : 0;
            tn = lp < nl ? (int)L[lp] : 0x7fffffff;
        }
        if (!wactive) continue;
        const int rs = (e0 - rbeg) * JMAX, re = rs + nent * JMAX;
        auto rank = [&](int tl) { return __float_as_int(sm.eoff[tl / JMAX].w) + tl % JMAX; };
        // this lane's next entry of the round that this row owns (j above i; a parity rule that
        // balances the owned counts, owner i iff (i + j even) == (i < j), measured 18.6 ms on c4)
        auto skip = [&]() {
            while (tn < re && rank(tn - rs) <= ki) {
                lp += S;
                tn = lp < nl ? (int)L[lp] : 0x7fffffff;
            }
        };
        skip();
#pragma unroll 1
        while (__any_sync(0xffffffffu, tn < re)) {
            if (tn < re) {
                const int tl = tn - rs;
                const int j = rank(tl);
                const float4 jp = sm.raw[tl];
                const float4* pay = sm.pay + tl * 9;
                float4 Q[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) Q[t] = pay[t];
                const float imj = 1.f / pay[8].z;
                const float2 x01 = __fadd2_rn(make_float2(ix, iy), make_float2(-jp.x, -jp.y));  // x_ij, exact (O1)
                const float x2 = iz - jp.z;
                const float r2 = s32_of(x01.x, x01.y, x2);
                const AccTerms T = acc_terms(Ri, Q, jp.w, x01, x2, r2, A.Cl, A.Cq, A.e2);
                const float VV = Ri[7].x * Q[7].x;
                const float f = VV * T.PQ;   // F = V_i V_j (P_i + P_j + Q) G: m_i dv_i -= F, m_j dv_j += F
                const float vg = VV * T.vG;
                s01 = __ffma2_rn(make_float2(-f, -f), T.G01, s01);
                s2 = fmaf(-f, T.G2, s2);
                s3 = fmaf(Ri[7].y + T.Qh, vg, s3);  // m_i du_i/dt += V_i V_j (P_i + Q/2) v_ij.G
                const float fj = f * imj;
                red_add_v4(A.acc + j, fj * T.G01.x, fj * T.G01.y, fj * T.G2, (Q[7].y + T.Qh) * vg * imj);
                lp += S;
                tn = lp < nl ? (int)L[lp] : 0x7fffffff;
                skip();
            }
        }
    }
    if (wactive) {
        s01.x = slot_sum<-S>(s01.x); s01.y = slot_sum<-S>(s01.y); s2 = slot_sum<-S>(s2); s3 = slot_sum<-S>(s3);
        const float imi = 1.f / Ri[8].z;
        if (ivalid && sl == 0) red_add_v4(A.acc + ki, s01.x * imi, s01.y * imi, s2 * imi, s3 * imi);
    }
}

__global__ void k_acc_finish(int64_t ng, const float4* __restrict__ acc, const int32_t* __restrict__ gas_idx, float dt,
                             float* ahx, float* ahy, float* ahz, float* dudt, float* vx, float* vy, float* vz,
                             float* u, const int32_t* gate = nullptr) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ng || (gate && *gate != 0)) return;
    const float4 q = acc[k];
    const int64_t i = gas_idx[k];
    if (ahx) { ahx[i] = q.x; ahy[i] = q.y; ahz[i] = q.z; }
    if (dudt) dudt[i] = q.w;
    if (dt != 0.f) {
        vx[i] = fmaf(dt, q.x, vx[i]);
        vy[i] = fmaf(dt, q.y, vy[i]);
        vz[i] = fmaf(dt, q.z, vz[i]);
        u[i] = fmaf(dt, q.w, u[i]);
    }
}

// ============================================================== smoothing-length update (NEXT-2)
// H_i' = factor * sqrt(d2_(k)), d2_(k) the k-th smallest s32 (the O2 fp32 squared distance)
// to another gas particle, selected among i's neighbour list.  The list holds every gas j
// with s32 < H_i^2, so the selection is exact when d2_(k) < H_i^2; otherwise (the k-th
// neighbour moved out, or fewer than k entries) H_i' is an upper bound / a doubling and i
// is counted as unconverged: rebuild the lists with H' and update again.
__global__ void __launch_bounds__(64) k_update_h(RowView rv, ListView lv, const float4* __restrict__ gpos,
                                                 const int32_t* __restrict__ gas_idx, int kth, float factor,
                                                 float* H_out, int* n_unconverged) {
    const int a = blockIdx.x;
    const int ii = threadIdx.x;
    const int icount = rv.icount[a];
    if (ii >= icount) return;
    const int ki = rv.ifirst[a] + ii;
    const int rbeg = rv.row_off[a];
    const float4 pi = gpos[ki];
    const float h2i = __fmul_rn(pi.w, pi.w);
    const int ntrue = lv.ncnt[ki];
    const bool row_lists = (rv.row_end[a] - rbeg) * JMAX <= 65536;  // longer rows have no lists
    const int nl = row_lists ? min(ntrue, lv.cap) : 0;
    const uint16_t* L = lv.nbr + (int64_t)ki * lv.cap;
    float d2[128];
    int m = 0;
    for (int p = 0; p < nl && m < 128; ++p) {
        const int t = L[p];
        int first, count, leaf, code;
        unpack_entry(__ldg(rv.erec + rbeg + t / JMAX), first, count, leaf, code);
        const int j = first + t % JMAX;
        if (j == ki) continue;
        int sx, sy, sz;
        decode_shift(code, sx, sy, sz);
        const float4 pj = gpos[j];
        const float dx = (pj.x + (float)sx * rv.L[0]) - pi.x;  // exact (O1)
        const float dy = (pj.y + (float)sy * rv.L[1]) - pi.y;
        const float dz = (pj.z + (float)sz * rv.L[2]) - pi.z;
        d2[m++] = s32_of(dx, dy, dz);
    }
    float sel = INFINITY;
    for (int c = 0; c < m; ++c) {  // the k-th smallest: #{< v} < k <= #{<= v}
        const float v = d2[c];
        int lt = 0, le = 0;
        for (int e = 0; e < m; ++e) {
            lt += d2[e] < v;
            le += d2[e] <= v;
        }
        if (lt < kth && kth <= le) { sel = v; break; }
    }
    // exact iff the list is complete and the k-th neighbour lies inside H_i; a truncated list
    // gives an upper bound (its k-th is >= the true one); too few entries grow H (volume x2),
    // a row without lists shrinks it
    const bool complete = row_lists && ntrue <= lv.cap;
    const bool exact = complete && sel < h2i;
    float Hn;
    if (!row_lists) Hn = 0.9f * pi.w;
    else if (sel < INFINITY) Hn = __fmul_rn(factor, __fsqrt_rn(sel));
    else Hn = 1.26f * pi.w;
    if (!exact) atomicAdd(n_unconverged, 1);
    H_out[gas_idx[ki]] = Hn;
}

// ============================================================== launches
// sel: the passes that honour crk_select_rows (corrections, extras, accel/du-dt); geometry and
// the count passes always cover every row
static RowView hydro_rows(crk_ctx* c, bool sel = false) {
    RowView rv;
    rv.ifirst = P<int32_t>(c->lfirst[2]);
    rv.icount = P<int32_t>(c->lcount[2]);
    rv.row_off = P<int32_t>(c->rowoff[1]);
    rv.row_end = P<int32_t>(c->rowend[1]);
    rv.erec = P<int2>(c->erec[1]);
    rv.box8 = P<float4>(c->lbox8[3]);
    for (int a = 0; a < 3; ++a) rv.L[a] = c->lay.L[a];
    rv.rclass = P<uint8_t>(c->rclass);
    rv.rsel = sel ? c->row_sel : 0;
    return rv;
}

template <class Pass, int ENT, int MINB = 1, int NW = HYD_NW, int G = HYD_G>
static crk_status launch_hyd(crk_ctx* c, const Pass& ps, cudaStream_t st, const char* what, bool sel = false) {
    if (c->nleaf[2] == 0) return CRK_OK;
    static_assert(NW * G >= 64, "a CTA covers a whole gas i-leaf (<= 64)");
    CRK_TRY(cuda_check(c, launch_pairs<Pass, NW, G, ENT, MINB>(ps, hydro_rows(c, sel), c->nleaf[2], st), what));
    c->launches++;
    return CRK_OK;
}


static void common(crk_ctx* c, HydCommon& h) {
    h.gpos = P<float4>(c->gpos);
    h.gas_idx = P<int32_t>(c->gas_idx);
}

static ListView list_view(crk_ctx* c) {
    ListView lv;
    lv.nbr = P<uint16_t>(c->nbr);
    lv.ncnt = P<int32_t>(c->ncnt);
    lv.lflag = P<uint32_t>(c->lflag);
    lv.frows = P<int32_t>(c->lflag) + c->nleaf[2];
    lv.nfrows = P<int32_t>(c->lflag) + 2 * c->nleaf[2];
    lv.cap = c->nbr_cap;
    lv.nrows = (int)c->nleaf[2];
    lv.work = P<int>(c->work) + 4;
    return lv;
}
static bool lists_on(crk_ctx* c) { return c->nbr_cap > 0 && c->nleaf[2] > 0; }

// list-driven launch of a gather/accel pass, then the on-the-fly kernel over the rows whose
// lists are incomplete (flagged by the builder; usually none: those CTAs exit at once)
template <class Pass, int ENT, int MINB, int FENT, int FMINB, int LG = HYD_G, bool SL = false>
static crk_status launch_listed(crk_ctx* c, const Pass& ps, cudaStream_t st, const char* what) {
    if (c->nleaf[2] == 0) return CRK_OK;
    RowView rv = hydro_rows(c, true);
    CRK_TRY(grow(c, c->work, 64, st));
    CRK_TRY(cuda_check(c, (launch_list<Pass, HYD_NW, LG, ENT, MINB, SL>(ps, rv, list_view(c), st)), what));
    c->launches++;
    const ListView lv = list_view(c);
    rv.rows = lv.frows;
    rv.nrows = lv.nfrows;
    CRK_TRY(cuda_check(c, launch_pairs<Pass, HYD_NW, HYD_G, FENT, FMINB>(ps, rv, c->nleaf[2], st), what));
    c->launches++;
    return CRK_OK;
}

crk_status geometry(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    if (lists_on(c)) {
        GeoPass<false, true> g;
        common(c, g);
        g.jrows = P<float4>(c->gpos);
        g.jpay = nullptr;
        g.gV = P<float>(c->gV);
        g.gposV = P<float4>(c->gposV);
        g.Vout = p->V;
        g.cnt = nullptr;
        const int64_t ng = c->n_gas > 0 ? c->n_gas : 1;
        CRK_TRY(grow(c, c->nbr, (size_t)ng * c->nbr_cap * sizeof(uint16_t), st));
        CRK_TRY(grow(c, c->ncnt, (size_t)ng * sizeof(int32_t) + 64, st));  // + pad: 16-byte-aligned bulk reads
        // lflag: per-row flags, then the compact flagged-row list, then its length
        const size_t fl = (size_t)(2 * c->nleaf[2] + 1) * sizeof(int32_t);
        CRK_TRY(grow(c, c->lflag, fl, st));
        CRK_TRY(cuda_check(c, zero_async(c->lflag.p, fl, st, c), "memset"));
        g.lv = list_view(c);
        return launch_hyd<GeoPass<false, true>, 128, 4>(c, g, st, "geometry (list build) kernel");
    }
    GeoPass<false> g;
    common(c, g);
    g.jrows = P<float4>(c->gpos);
    g.jpay = nullptr;
    g.gV = P<float>(c->gV);
    g.gposV = P<float4>(c->gposV);
    g.Vout = p->V;
    g.cnt = nullptr;
    return launch_hyd<GeoPass<false>, 128, 2>(c, g, st, "geometry kernel");
}

static CorPass cor_pass(crk_ctx* c, crk_particles* p) {
    CorPass g;
    common(c, g);
    g.jrows = P<float4>(c->gposV);
    g.jpay = nullptr;
    g.gcoef = P<float>(c->gcoef);
    g.ng = c->n_gas;
    g.A = p->A; g.B = p->B; g.dA = p->dA; g.dB = p->dB;
    g.n = c->n;
    return g;
}

crk_status corrections(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    CorPass g = cor_pass(c, p);
    if (lists_on(c)) return launch_listed<CorPass, 128, 3, 128, 3>(c, g, st, "corrections kernel");
    return launch_hyd<CorPass, 128, 3>(c, g, st, "corrections kernel", true);
}

__global__ void k_gather_gas_state(int64_t ng, const int32_t* gas_idx, const float* vx, const float* vy,
                                   const float* vz, const float* m, const float* u, float4* gvel, float* gu) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ng) return;
    const int64_t i = gas_idx[k];
    gvel[k] = make_float4(vx[i], vy[i], vz[i], m[i]);
    gu[k] = u[i];
}

static crk_status gather_gas_state(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    k_gather_gas_state<<<(unsigned)((c->n_gas + 255) / 256), 256, 0, st>>>(
        c->n_gas, P<int32_t>(c->gas_idx), p->vx, p->vy, p->vz, p->m, p->u, P<float4>(c->gvel), P<float>(c->gu));
    CRK_LAUNCHED(c, "gather gas state");
    return CRK_OK;
}

static ExtPass ext_pass(crk_ctx* c, crk_particles* p) {
    ExtPass g;
    common(c, g);
    g.jrows = P<float4>(c->gposV);
    g.jpay = P<float4>(c->gvel);
    g.gV = P<float>(c->gV);
    g.gcoef = P<float>(c->gcoef);
    g.gvel = P<float4>(c->gvel);
    g.gu = P<float>(c->gu);
    g.grec = P<float4>(c->grec);
    g.ng = c->n_gas;
    g.n = c->n;
    g.gamma = c->prm.gamma;
    g.rho = p->rho; g.P = p->P; g.cs = p->cs; g.dv = p->dv;
    return g;
}

crk_status extras(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    if (c->n_gas == 0) return CRK_OK;
    CRK_TRY(gather_gas_state(c, p, st));
    ExtPass g = ext_pass(c, p);
    if (lists_on(c)) return launch_listed<ExtPass, 128, 3, 128, 3>(c, g, st, "extras kernel");
    return launch_hyd<ExtPass, 128, 3>(c, g, st, "extras kernel", true);
}

// a5 + a6 fused: one list kernel walks each i's list twice (Corrections, then Extras with
// the coefficients just computed), sharing the row staging; flagged rows run the on-the-fly
// Corrections then Extras kernels over the flagged-row list.
crk_status corrections_extras(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    if (!lists_on(c)) {
        CRK_TRY(corrections(c, p, st));
        return extras(c, p, st);
    }
    CRK_TRY(gather_gas_state(c, p, st));
    if (c->prm.hydro_kernel == 2) {  // one list walk (CorExtPass), on-the-fly kernel for flagged rows
        CorExtPass g;
        common(c, g);
        g.jrows = P<float4>(c->gposV);
        g.jpay = P<float4>(c->gvel);
        g.gV = P<float>(c->gV);
        g.gvel = P<float4>(c->gvel);
        g.gu = P<float>(c->gu);
        g.grec = P<float4>(c->grec);
        g.ng = c->n_gas;
        g.n = c->n;
        g.gamma = c->prm.gamma;
        g.A = p->A; g.B = p->B; g.dA = p->dA; g.dB = p->dB;
        g.rho = p->rho; g.P = p->P; g.cs = p->cs; g.dv = p->dv;
        return launch_listed<CorExtPass, 128, 2, 128, 2>(c, g, st, "corrections + extras (one walk) kernel");
    }
    const CorPass gc = cor_pass(c, p);
    const ExtPass ge = ext_pass(c, p);
    RowView rv = hydro_rows(c, true);
    const ListView lv = list_view(c);
    // the row's lists staged in shared memory while 4 CTAs per SM still fit (cap <= 160)
    CRK_TRY(cuda_check(c, (launch_list2<CorPass, ExtPass, HYD_NW, HYD_G, 128, 4>(gc, ge, rv, lv, st,
                                                                                lv.cap <= 160)),
                       "corrections + extras kernel"));
    c->launches++;
    rv.rows = lv.frows;
    rv.nrows = lv.nfrows;
    CRK_TRY(cuda_check(c, (launch_pairs<CorPass, HYD_NW, HYD_G, 128, 3>(gc, rv, c->nleaf[2], st)), "corrections kernel"));
    CRK_TRY(cuda_check(c, (launch_pairs<ExtPass, HYD_NW, HYD_G, 128, 3>(ge, rv, c->nleaf[2], st)), "extras kernel"));
    c->launches += 2;
    return CRK_OK;
}

// symmetric accel over the lists (acc_symlist_kernel); if any row is flagged the symmetric
// kernel and its finish exit on the device and the gated i-centric list kernels run instead
static crk_status accel_symlist(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    const int64_t ng = c->n_gas;
    CRK_TRY(grow(c, c->gacc, (ng > 0 ? ng : 1) * 16, st));
    CRK_TRY(cuda_check(c, zero_async(c->gacc.p, (ng > 0 ? ng : 1) * 16, st, c), "memset"));
    CRK_TRY(grow(c, c->work, 64, st));
    AccSymListArgs A;
    A.gpos = P<float4>(c->gpos);
    A.grec = P<float4>(c->grec);
    A.rv = hydro_rows(c, true);
    A.lv = list_view(c);
    A.acc = P<float4>(c->gacc);
    A.ng = c->n_gas;
    A.Cl = c->prm.av_cl; A.Cq = c->prm.av_cq; A.e2 = c->prm.av_eps2;
    const int smem = ASL_LIST_OFF + ASL_NW * ASL_G * c->nbr_cap * (int)sizeof(uint16_t);
    cudaError_t e = cudaFuncSetAttribute(acc_symlist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_check(c, e, "smem attribute");
    if (A.lv.nrows > 0) acc_symlist_kernel<<<A.lv.nrows, ASL_NW * 32, smem, st>>>(A);
    CRK_LAUNCHED(c, "accel/dudt (symmetric list) kernel");
    k_acc_finish<<<(unsigned)((ng + 255) / 256), 256, 0, st>>>(ng, P<float4>(c->gacc), P<int32_t>(c->gas_idx), dt,
                                                               p->ahx, p->ahy, p->ahz, p->dudt, p->vx, p->vy, p->vz,
                                                               p->u, A.lv.nfrows);
    CRK_LAUNCHED(c, "accel finish");
    // flagged rows present: i-centric list kernel (gated) + on-the-fly kernel over the flagged rows
    AccPass<false, 32> g;
    common(c, g);
    g.jrows = P<float4>(c->gpos);
    g.jpay = P<float4>(c->grec);
    g.grec = P<float4>(c->grec);
    g.Cl = c->prm.av_cl; g.Cq = c->prm.av_cq; g.e2 = c->prm.av_eps2; g.dt = dt;
    g.n = c->n;
    g.ng = c->n_gas;
    g.ahx = p->ahx; g.ahy = p->ahy; g.ahz = p->ahz; g.dudt = p->dudt;
    g.vx = p->vx; g.vy = p->vy; g.vz = p->vz; g.u = p->u;
    g.cnt = nullptr;
    ListView lv = list_view(c);
    lv.gate = 1;
    RowView rv = hydro_rows(c, true);
    CRK_TRY(cuda_check(c, launch_list<AccPass<false, 32>, HYD_NW, HYD_G, 72, 2>(g, rv, lv, st), "accel/dudt kernel"));
    c->launches++;
    rv.rows = lv.frows;
    rv.nrows = lv.nfrows;
    CRK_TRY(cuda_check(c, launch_pairs<AccPass<false, 32>, HYD_NW, HYD_G, 72, 2>(g, rv, c->nleaf[2], st), "accel/dudt kernel"));
    c->launches++;
    return CRK_OK;
}

template <int BT, int ENT>
static crk_status accel_gather(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    AccPass<false, BT> g;
    common(c, g);
    g.jrows = P<float4>(c->gpos);
    g.jpay = P<float4>(c->grec);
    g.grec = P<float4>(c->grec);
    g.Cl = c->prm.av_cl; g.Cq = c->prm.av_cq; g.e2 = c->prm.av_eps2; g.dt = dt;
    g.n = c->n;
    g.ng = c->n_gas;
    g.ahx = p->ahx; g.ahy = p->ahy; g.ahz = p->ahz; g.dudt = p->dudt;
    g.vx = p->vx; g.vy = p->vy; g.vz = p->vz; g.u = p->u;
    g.cnt = nullptr;
    // (16 lanes per i, G = 2, measured slower on c4: 15.8 vs 12.3 ms — a list's consecutive entries
    // are 68 of the row's 512 slots, so their bank groups are no less random than 8 i's runs)
    // the row's lists staged in shared memory (rounds of 64 entries: 99.5% of the c4 rows are one
    // round) while two CTAs per SM still fit (cap <= 144); else rounds of 72 and global list reads
    if (lists_on(c) && c->nbr_cap <= 144 && c->nbr_cap % 8 == 0)
        return launch_listed<AccPass<false, BT>, 64, 2, ENT, 2, HYD_G, true>(c, g, st, "accel/dudt kernel");
    if (lists_on(c)) return launch_listed<AccPass<false, BT>, 72, 2, ENT, 2>(c, g, st, "accel/dudt kernel");
    return launch_hyd<AccPass<false, BT>, ENT, 2>(c, g, st, "accel/dudt kernel");
}

// experiment (crk_params.hydro_kernel = 4 / 6): 8 lanes per i (4 i per warp, 16 warps per CTA, one
// CTA per SM): a quarter-warp then reads one i's consecutive slots (no bank conflicts between
// two i's) at the cost of the overlap between two CTAs' staging
template <int ENT>
static crk_status accel_s8(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    if (!lists_on(c)) return accel_gather<32, 72>(c, p, dt, st);
    AccPass<false, 32> g;
    common(c, g);
    g.jrows = P<float4>(c->gpos);
    g.jpay = P<float4>(c->grec);
    g.grec = P<float4>(c->grec);
    g.Cl = c->prm.av_cl; g.Cq = c->prm.av_cq; g.e2 = c->prm.av_eps2; g.dt = dt;
    g.n = c->n;
    g.ng = c->n_gas;
    g.ahx = p->ahx; g.ahy = p->ahy; g.ahz = p->ahz; g.dudt = p->dudt;
    g.vx = p->vx; g.vy = p->vy; g.vz = p->vz; g.u = p->u;
    g.cnt = nullptr;
    if (c->nleaf[2] == 0) return CRK_OK;
    RowView rv = hydro_rows(c, true);
    CRK_TRY(grow(c, c->work, 64, st));
    CRK_TRY(cuda_check(c, (launch_list<AccPass<false, 32>, 16, 4, ENT, 1>(g, rv, list_view(c), st)), "accel/dudt kernel"));
    c->launches++;
    const ListView lv = list_view(c);
    rv.rows = lv.frows;
    rv.nrows = lv.nfrows;
    CRK_TRY(cuda_check(c, (launch_pairs<AccPass<false, 32>, HYD_NW, HYD_G, 72, 2>(g, rv, c->nleaf[2], st)),
                       "accel/dudt kernel"));
    c->launches++;
    return CRK_OK;
}

crk_status accel_dudt(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    if (dt != 0.f && (!p->vx || !p->vy || !p->vz || !p->u)) return fail(c, CRK_EINVAL, "kick needs v and u");
    // opt-in (hydro_kernel = 5): c4 14.9 ms vs 12.3 for the i-centric list kernel (the per-pair
    // red.global reactions cost more than the halved pair work saves)
    if (lists_on(c) && !c->lay.partial && c->row_sel == 0 && c->prm.hydro_kernel == 5 && c->nbr_cap % 8 == 0 &&
        c->nbr_cap <= 256)
        return accel_symlist(c, p, dt, st);
    switch (c->prm.hydro_kernel) {
        case 4: return accel_s8<72>(c, p, dt, st);
        case 6: return accel_s8<128>(c, p, dt, st);
        default: return accel_gather<32, 72>(c, p, dt, st);
    }
}

crk_status hydro_count(crk_ctx* c, int32_t* cgather, int32_t* csym, cudaStream_t st) {
    if (lists_on(c) && c->stage >= ST_GEO) {  // the walks corrections/extras and accel/du-dt make
        ListCountPass<false> g;
        common(c, g);
        g.jrows = P<float4>(c->gpos);
        g.jpay = nullptr;
        g.cnt = cgather;
        CRK_TRY((launch_listed<ListCountPass<false>, 128, 3, 128, 3>(c, g, st, "gather count (list walk)")));
        ListCountPass<true> a;
        common(c, a);
        a.jrows = P<float4>(c->gpos);
        a.jpay = nullptr;
        a.cnt = csym;
        return launch_listed<ListCountPass<true>, 128, 3, 128, 3>(c, a, st, "sym count (list walk)");
    }
    GeoPass<true> g;
    common(c, g);
    g.jrows = P<float4>(c->gpos);
    g.jpay = nullptr;
    g.gV = nullptr; g.gposV = nullptr; g.Vout = nullptr; g.cnt = cgather;
    CRK_TRY((launch_hyd<GeoPass<true>, 128>(c, g, st, "gather count kernel")));
    AccPass<true> a;
    common(c, a);
    a.jrows = P<float4>(c->gpos);
    a.jpay = nullptr;
    a.grec = nullptr;
    a.cnt = csym;
    return launch_hyd<AccPass<true>, 128>(c, a, st, "sym count kernel");
}

// crk_neighbour_lists: the geometry-built lists decoded to sorted positions (one CTA per gas
// i-leaf, one thread per member)
__global__ void __launch_bounds__(64) k_decode_lists(RowView rv, ListView lv, const int32_t* __restrict__ gas_idx,
                                                    int cap_out, int32_t* count, int32_t* nbr) {
    const int a = blockIdx.x;
    const int ii = threadIdx.x;
    if (ii >= rv.icount[a]) return;
    const int k = rv.ifirst[a] + ii;
    const int rbeg = rv.row_off[a];
    const bool row_lists = (rv.row_end[a] - rbeg) * JMAX <= 65536;
    const int ntrue = lv.ncnt[k];
    const bool complete = row_lists && !lv.lflag[a] && ntrue <= lv.cap;
    const int64_t i = gas_idx[k];
    count[i] = complete ? ntrue : -1;
    if (!complete) return;
    const uint16_t* L = lv.nbr + (int64_t)k * lv.cap;
    const int m = min(ntrue, cap_out);
    for (int t = 0; t < m; ++t) {
        const int slot = L[t];
        int first, cnt, leaf, code;
        unpack_entry(__ldg(rv.erec + rbeg + slot / JMAX), first, cnt, leaf, code);
        nbr[i * cap_out + t] = gas_idx[first + slot % JMAX];
    }
}

crk_status neighbour_lists(crk_ctx* c, int32_t cap_out, int32_t* count, int32_t* nbr, cudaStream_t st) {
    CRK_TRY(cuda_check(c, zero_async(count, (size_t)c->n * 4, st, c), "memset"));
    if (c->nleaf[2] == 0) return CRK_OK;
    k_decode_lists<<<(unsigned)c->nleaf[2], 64, 0, st>>>(hydro_rows(c), list_view(c), P<int32_t>(c->gas_idx),
                                                         cap_out, count, nbr);
    CRK_LAUNCHED(c, "decode neighbour lists");
    return CRK_OK;
}

crk_status update_h(crk_ctx* c, int kth, float factor, float* H_out, int32_t* n_unconverged, cudaStream_t st) {
    if (!lists_on(c)) return fail(c, CRK_ESTATE, "update_h needs the neighbour lists (crk_params.nbr_cap >= 0)");
    CRK_TRY(cuda_check(c, zero_async(n_unconverged, sizeof(int32_t), st, c), "memset"));
    k_update_h<<<(unsigned)c->nleaf[2], 64, 0, st>>>(hydro_rows(c), list_view(c), P<float4>(c->gpos),
                                                     P<int32_t>(c->gas_idx), kth, factor, H_out, n_unconverged);
    CRK_LAUNCHED(c, "update H");
    return CRK_OK;
}

}  // namespace crk
