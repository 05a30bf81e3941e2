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

// ============================================================== symmetric (Newton-3) variant
// Each unordered pair {i, j} is evaluated once, by the warp of the lower i-group.
// gkey[j] = sorted index of the first particle of j's group (warp w of gravity i-leaf a
// covers [first_a + 16w, first_a + 16w + 16)), so group order is a total order.  Lanes
// own the j-survivors and loop over the warp's 16 i-particles (shared-memory
// broadcast); the i-side sums stay in registers for the whole row and are reduced
// once at the end; the j-side reactions (and the final i-side sums) go to a float4
// accumulator with red.global.add.v4.f32 — the set of terms is fixed, their summation
// order depends on scheduling.  Within the own group the pair is met from both sides,
// so there only the survivor's (j-side) half is accumulated.  Survivors carry over
// across chunks so that every warp step but the last is full.
namespace symg {
constexpr int NW = 8, G = 16, CH = 256, CAP = CH + 32;
struct Smem {
    float4 jpos[CH];
    int jg[CH];
    int jidx[CH];
    float4 elo[CH / JMAX], ehi[CH / JMAX];
    float4 ipos[NW][G];
    float4 wpos[NW][CAP];
    int widx[NW][CAP];
    uint8_t went[NW][32];
};
}  // namespace symg

__device__ __forceinline__ void red_add_v4(float4* p, float a, float b, float c) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(0.f)
                 : "memory");
}

struct GravSymArgs {
    const float4* xm;
    const int32_t* gkey;
    float4* acc;
    float rcut2, eps2;
    float c0, c1, c2, c3, c4, c5;
};

__global__ void __launch_bounds__(symg::NW * 32, 2) grav_sym_kernel(const GravSymArgs A, const RowView rv) {
    using namespace symg;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int a = blockIdx.x;
    const int ifirst = rv.ifirst[a];
    const int icount = rv.icount[a];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ibase = warp * G;
    const bool wactive = ibase < icount;
    const int gself = ifirst + ibase;  // this warp's group key
    const int ng = min(G, icount - ibase);

    float lo[3] = {0.f, 0.f, 0.f}, hi[3] = {0.f, 0.f, 0.f};
    const float wcut = A.rcut2 * CULL_SLACK;
    if (wactive) {
        const bool iv = lane < ng;
        float4 p = make_float4(-1e18f, -1e18f, -1e18f, 0.f);  // far sentinel: finite products
        if (iv) p = A.xm[gself + lane];
        if (lane < G) sm.ipos[warp][lane] = p;
        lo[0] = warp_min(iv ? p.x : INFINITY);
        lo[1] = warp_min(iv ? p.y : INFINITY);
        lo[2] = warp_min(iv ? p.z : INFINITY);
        hi[0] = warp_max(iv ? p.x : -INFINITY);
        hi[1] = warp_max(iv ? p.y : -INFINITY);
        hi[2] = warp_max(iv ? p.z : -INFINITY);
    }
    float ax[G], ay[G], az[G];
#pragma unroll
    for (int i = 0; i < G; ++i) ax[i] = ay[i] = az[i] = 0.f;
    float4* wpos = sm.wpos[warp];
    int* widx = sm.widx[warp];
    uint8_t* went = sm.went[warp];
    const float rc2 = A.rcut2, e2 = A.eps2;
    const float c0 = A.c0, c1 = A.c1, c2 = A.c2, c3 = A.c3, c4 = A.c4, c5 = A.c5;

    // one warp step: lane owns survivor k0 + lane (or the far sentinel), loops over the group
    auto eval_step = [&](int k0, int kend) {
        const int k = k0 + lane;
        float4 jp = make_float4(1e18f, 1e18f, 1e18f, 0.f);
        int j = -1;
        if (k < kend) {
            jp = wpos[k];
            j = widx[k];
        }
        const float mj = j < 0 ? 0.f : (j & 0x40000000 ? 0.f : jp.w);  // own group: j-side only
        j &= 0x3fffffff;
        float bx = 0.f, by = 0.f, bz = 0.f;
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const float4 ip = sm.ipos[warp][i];
            const float dx = jp.x - ip.x, dy = jp.y - ip.y, dz = jp.z - ip.z;  // x_j - x_i
            const float r2 = s32_of(dx, dy, dz);
            const float ri = rsqrtf(r2 + e2);
            const float ri3 = ri * ri * ri;
            const float p5 = fmaf(fmaf(fmaf(fmaf(fmaf(c5, r2, c4), r2, c3), r2, c2), r2, c1), r2, c0);
            const float w = r2 < rc2 ? ri3 - p5 : 0.f;
            const float wi = mj * w;  // i-side: a_i += m_j w x_ji
            ax[i] = fmaf(wi, dx, ax[i]);
            ay[i] = fmaf(wi, dy, ay[i]);
            az[i] = fmaf(wi, dz, az[i]);
            const float wj = ip.w * w;  // j-side: a_j += m_i w x_ij
            bx = fmaf(-wj, dx, bx);
            by = fmaf(-wj, dy, by);
            bz = fmaf(-wj, dz, bz);
        }
        if (k < kend) red_add_v4(A.acc + j, bx, by, bz);
    };

    int cnt = 0;  // survivors waiting in the warp buffer
    const int rbeg = rv.row_off[a], rend = rv.row_off[a + 1];
    constexpr int EPC = CH / JMAX;
    const int nch = (rend - rbeg + EPC - 1) / EPC;
    for (int c = 0; c < nch; ++c) {
        const int nent = (rend - rbeg - c + nch - 1) / nch;
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
                const float4 p = __ldg(A.xm + j);
                sm.jpos[t] = make_float4(p.x + ox, p.y + oy, p.z + oz, p.w);
                sm.jg[t] = __ldg(A.gkey + j);
                sm.jidx[t] = j;
            } else {
                sm.jpos[t] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
                sm.jg[t] = -1;
            }
            if (k == 0 && m < nent) {
                const float* bb = rv.jbbox + 6 * (int64_t)b;
                sm.elo[m] = make_float4(__ldg(bb) + ox, __ldg(bb + 1) + oy, __ldg(bb + 2) + oz, 0.f);
                sm.ehi[m] = make_float4(__ldg(bb + 3) + ox, __ldg(bb + 4) + oy, __ldg(bb + 5) + oz, 0.f);
            }
        }
        __syncthreads();
        if (wactive) {
            bool ek = false;
            if (lane < nent) {
                const float4 bl = sm.elo[lane], bh = sm.ehi[lane];
                const float gx = fmaxf(fmaxf(bl.x - hi[0], lo[0] - bh.x), 0.f);
                const float gy = fmaxf(fmaxf(bl.y - hi[1], lo[1] - bh.y), 0.f);
                const float gz = fmaxf(fmaxf(bl.z - hi[2], lo[2] - bh.z), 0.f);
                ek = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) < wcut;
            }
            const unsigned em = __ballot_sync(0xffffffffu, ek);
            if (ek) went[__popc(em & ((1u << lane) - 1u))] = (uint8_t)lane;
            const int nsurv = __popc(em);
            __syncwarp();
            for (int q0 = 0; q0 < nsurv; q0 += 32 / JMAX) {
                const int qe = q0 + lane / JMAX;
                const int t = (qe < nsurv ? went[qe] : 0) * JMAX + lane % JMAX;
                const float4 p = sm.jpos[t];
                const int jgk = sm.jg[t];
                // pairs owned by this group: j in a later group, or j in this group
                const bool keep = qe < nsurv && jgk >= gself && box_dist2(p.x, p.y, p.z, lo, hi) < wcut;
                const unsigned msk = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int o = cnt + __popc(msk & ((1u << lane) - 1u));
                    wpos[o] = p;
                    widx[o] = sm.jidx[t] | (jgk == gself ? 0x40000000 : 0);
                }
                cnt += __popc(msk);
            }
            __syncwarp();
            const int nfull = cnt & ~31;
            for (int k0 = 0; k0 < nfull; k0 += 32) eval_step(k0, nfull);
            // move the remainder (< 32) to the front of the buffer
            const int rem = cnt - nfull;
            float4 rp;
            int ri = 0;
            if (nfull > 0 && lane < rem) {
                rp = wpos[nfull + lane];
                ri = widx[nfull + lane];
            }
            __syncwarp();
            if (nfull > 0 && lane < rem) {
                wpos[lane] = rp;
                widx[lane] = ri;
            }
            cnt = rem;
            __syncwarp();
        }
        __syncthreads();
    }
    if (wactive) {
        if (cnt > 0) eval_step(0, cnt);
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const float sx = warp_sum(ax[i]), sy = warp_sum(ay[i]), sz = warp_sum(az[i]);
            if (lane == i && i < ng) red_add_v4(A.acc + gself + i, sx, sy, sz);
        }
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

// group keys: gkey[k] = first_a + 16 ((k - first_a) / 16) for k in gravity i-leaf a
__global__ void k_group_keys(int64_t nl, const int32_t* __restrict__ first, const int32_t* __restrict__ count,
                             int32_t* gkey) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= nl) return;
    const int f = first[l], c = count[l];
    for (int t = 0; t < c; ++t) gkey[f + t] = f + symg::G * (t / symg::G);
}

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

static RowView grav_rows(crk_ctx* c) {
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
    return rv;
}

static crk_status gravity_sym(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    const int64_t n = c->n;
    CRK_TRY(grow(c, c->gacc, n * 16, st));
    CRK_TRY(grow(c, c->gkey, n * 4, st));
    CRK_TRY(cuda_check(c, cudaMemsetAsync(c->gacc.p, 0, n * 16, st), "memset"));
    if (c->nleaf[0] > 0) {
        k_group_keys<<<(unsigned)((c->nleaf[0] + 127) / 128), 128, 0, st>>>(
            c->nleaf[0], P<int32_t>(c->lfirst[0]), P<int32_t>(c->lcount[0]), P<int32_t>(c->gkey));
        CRK_LAUNCHED(c, "group keys");
        GravSymArgs A;
        A.xm = P<float4>(c->xm);
        A.gkey = P<int32_t>(c->gkey);
        A.acc = P<float4>(c->gacc);
        A.rcut2 = c->prm.rcut2;
        A.eps2 = c->prm.eps2;
        A.c0 = c->prm.poly[0]; A.c1 = c->prm.poly[1]; A.c2 = c->prm.poly[2];
        A.c3 = c->prm.poly[3]; A.c4 = c->prm.poly[4]; A.c5 = c->prm.poly[5];
        const int smem = (int)sizeof(symg::Smem);
        cudaError_t e = cudaFuncSetAttribute(grav_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_check(c, e, "smem attribute");
        grav_sym_kernel<<<(unsigned)c->nleaf[0], symg::NW * 32, smem, st>>>(A, grav_rows(c));
        CRK_LAUNCHED(c, "gravity (symmetric) kernel");
    }
    k_grav_finish<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, P<float4>(c->gacc), c->prm.G, dt, p->ax, p->ay,
                                                                p->az, p->vx, p->vy, p->vz);
    CRK_LAUNCHED(c, "gravity finish");
    return CRK_OK;
}

crk_status gravity_kick(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st) {
    if (dt != 0.f && (!p->vx || !p->vy || !p->vz)) return fail(c, CRK_EINVAL, "kick needs vx, vy, vz");
    if (c->prm.symmetric) return gravity_sym(c, p, dt, st);
    return launch_grav<false>(c, p, dt, nullptr, st);
}

crk_status gravity_count(crk_ctx* c, crk_particles* p, int32_t* cnt, cudaStream_t st) {
    return launch_grav<true>(c, p, 0.f, cnt, st);
}

}  // namespace crk
