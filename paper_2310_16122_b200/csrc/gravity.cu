// gravity.cu — a3: short-range gravity + kick.
//
//   a_i = G sum_{j != i, s32 < rcut2} m_j x_ji [ (s + eps2)^-3/2 - P5(s) ],  v_i += dt a_i
//
// Newtonian minus the fitted grid-force polynomial of order 5 (PAPER.md:147, 278,
// 646 HACC_CUDA_POLY_ORDER=5), Plummer-softened, inside the cutoff.  Per pair: one
// MUFU rsqrt and ~19 FP32 FMA-pipe instructions; FP32-ALU bound.
#include "pairs.cuh"

namespace crk {

template <bool COUNT>
struct GravPass {
    static constexpr int PAY = 0;
    static constexpr bool SYM = false;
    static constexpr int UNROLL = 4;
    const float4* xm;  // sorted (x, y, z, m)
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
    __device__ void stage(int j, float ox, float oy, float oz, float4& jp, float4*) const {
        const float4 p = __ldg(xm + j);
        jp = make_float4(p.x + ox, p.y + oy, p.z + oz, COUNT ? __int_as_float(j) : p.w);
    }
    __device__ __forceinline__ void pair(const I& s, Acc& a, const float4& jp, const float4*) const {
        const float dx = jp.x - s.x, dy = jp.y - s.y, dz = jp.z - s.z;  // exact (O1)
        const float r2 = s32_of(dx, dy, dz);
        if (COUNT) {
            a.n += (r2 < rcut2 && __float_as_int(jp.w) != s.idx) ? 1 : 0;
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
#pragma unroll
            for (int o = 16; o >= GG; o >>= 1) a.n += __shfl_xor_sync(0xffffffffu, a.n, o);
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

constexpr int GRAV_CH = 256;

template <bool COUNT>
static crk_status launch_grav(crk_ctx* c, crk_particles* p, float dt, int32_t* cnt, cudaStream_t st) {
    GravPass<COUNT> g;
    g.xm = P<float4>(c->xm);
    g.rcut2 = c->prm.rcut2;
    g.eps2 = c->prm.eps2;
    g.G = c->prm.G;
    g.dt = dt;
    g.c0 = c->prm.poly[0]; g.c1 = c->prm.poly[1]; g.c2 = c->prm.poly[2];
    g.c3 = c->prm.poly[3]; g.c4 = c->prm.poly[4]; g.c5 = c->prm.poly[5];
    g.ax = p->ax; g.ay = p->ay; g.az = p->az;
    g.vx = p->vx; g.vy = p->vy; g.vz = p->vz;
    g.cnt = cnt;
    RowView rv;
    rv.ifirst = P<int32_t>(c->lfirst[0]);
    rv.icount = P<int32_t>(c->lcount[0]);
    rv.jfirst = P<int32_t>(c->lfirst[1]);
    rv.jcount = P<int32_t>(c->lcount[1]);
    rv.row_off = P<int32_t>(c->rowoff[0]);
    rv.col = P<int32_t>(c->col[0]);
    rv.shift = P<int8_t>(c->shift[0]);
    rv.jbbox = P<float>(c->lbbox[1]);
    rv.jmaxh2 = nullptr;
    for (int a = 0; a < 3; ++a) rv.L[a] = c->lay.L[a];
    if (c->nleaf[0] == 0) return CRK_OK;
    pair_kernel<GravPass<COUNT>, GRAV_NW, GRAV_G, GRAV_CH, 1>
        <<<(unsigned)c->nleaf[0], GRAV_NW * 32, 0, st>>>(g, rv);
    CRK_LAUNCHED(c, "gravity kernel");
    return CRK_OK;
}

crk_status gravity_kick(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    if (dt != 0.f && (!p->vx || !p->vy || !p->vz)) return fail(c, CRK_EINVAL, "kick needs vx, vy, vz");
    return launch_grav<false>(c, p, dt, nullptr, st);
}

crk_status gravity_count(crk_ctx* c, crk_particles* p, int32_t* cnt, cudaStream_t st) {
    return launch_grav<true>(c, p, 0.f, cnt, st);
}

}  // namespace crk
