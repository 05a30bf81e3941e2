// integrate.cu — the steps either side of the short-range passes in a sub-cycle
// ("called more than once in a single timestep"):
// Courant / acceleration time-step limit (a grid-wide float minimum: the paper's float
// fetch_min, CAS-emulated on NVIDIA at PAPER.md:389, is here an integer atomicMin on the
// bits of non-negative floats), the kick v += dt a, u += dt du/dt, and the drift
// x += dt v kept on the position quantum q (O1).  Readings in DESIGN.md §2 ("Sub-cycle").
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace crk {

crk_status refresh(crk_ctx* c, crk_particles* p, cudaStream_t st);  // build.cu

__global__ void k_set_inf(float* dt) { *reinterpret_cast<int*>(dt) = 0x7f800000; }

// dt_i = C_acc sqrt(eps / |a_i|) for every particle (a = gravity + hydro for gas) and also
// C_cfl H_i / c_i for gas; out = min_i dt_i (atomicMin on the bits: dt_i >= 0)
__global__ void __launch_bounds__(256) k_courant(int64_t n, const uint8_t* __restrict__ species,
                                                 const int32_t* __restrict__ grank, const float4* __restrict__ grec,
                                                 const float* __restrict__ H, const float* ax, const float* ay,
                                                 const float* az, const float* ahx, const float* ahy,
                                                 const float* ahz, float eps, float c_cfl, float c_acc, float* out) {
    __shared__ float wmin[8];
    float best = INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float gx = ax[i], gy = ay[i], gz = az[i];
        const bool gas = species[i] == 1;
        if (gas) { gx += ahx[i]; gy += ahy[i]; gz += ahz[i]; }
        const float a = sqrtf(fmaf(gz, gz, fmaf(gy, gy, gx * gx)));
        float d = a > 0.f ? c_acc * sqrtf(eps / a) : INFINITY;
        if (gas) {
            const float c = grec[9 * (int64_t)grank[i] + 2].w;  // sound speed (Extras record)
            if (c > 0.f) d = fminf(d, c_cfl * H[i] / c);
        }
        best = fminf(best, d);
    }
    best = warp_min(best);
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? wmin[threadIdx.x] : INFINITY;
        v = warp_min(v);
        if (threadIdx.x == 0) atomicMin(reinterpret_cast<int*>(out), __float_as_int(v));
    }
}

__global__ void k_kick(int64_t n, const uint8_t* __restrict__ species, float dt, const float* ax, const float* ay,
                       const float* az, const float* ahx, const float* ahy, const float* ahz, const float* dudt,
                       float* vx, float* vy, float* vz, float* u) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float gx = ax[i], gy = ay[i], gz = az[i];
    if (species[i] == 1) {
        gx += ahx[i]; gy += ahy[i]; gz += ahz[i];
        u[i] = __fmaf_rn(dt, dudt[i], u[i]);
    }
    vx[i] = __fmaf_rn(dt, gx, vx[i]);
    vy[i] = __fmaf_rn(dt, gy, vy[i]);
    vz[i] = __fmaf_rn(dt, gz, vz[i]);
}

// x' = fl32(x + dt v) (one rounding), rounded to the nearest multiple of q (ties to even),
// wrapped into [0, L): every op exact except the fma (q and L are powers of two)
__device__ __forceinline__ float drift1(float x, float v, float dt, float inv_q, float q, float L, bool wrap) {
    const float t = __fmaf_rn(dt, v, x);
    float r = __fmul_rn(rintf(__fmul_rn(t, inv_q)), q);
    if (wrap) {
        if (r >= L) r = __fsub_rn(r, L);
        else if (r < 0.f) r = __fadd_rn(r, L);
    }
    return r;
}

// wrap = false (skin lists): positions may leave [0, L) by < skin/2; the largest |x' - x|
// (fp32 Euclidean, rounded up by 1 ulp) goes to *dmax (atomicMax on the bits, >= 0)
__global__ void k_drift(int64_t n, float dt, float inv_q, float q, float Lx, float Ly, float Lz, float* x, float* y,
                        float* z, const float* vx, const float* vy, const float* vz, bool wrap, float* dmax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x0 = x[i], y0 = y[i], z0 = z[i];
    const float x1 = drift1(x0, vx[i], dt, inv_q, q, Lx, wrap);
    const float y1 = drift1(y0, vy[i], dt, inv_q, q, Ly, wrap);
    const float z1 = drift1(z0, vz[i], dt, inv_q, q, Lz, wrap);
    x[i] = x1; y[i] = y1; z[i] = z1;
    if (!wrap) {
        const float dx = x1 - x0, dy = y1 - y0, dz = z1 - z0;
        const float d = nextafterf(sqrtf(fmaf(dz, dz, fmaf(dy, dy, dx * dx))), INFINITY);
        atomicMax(reinterpret_cast<int*>(dmax), __float_as_int(d));
    }
}

// bound since the build += this drift's largest displacement (a sum of maxima bounds every
// particle's total displacement)
__global__ void k_disp_accum(float* disp) {
    disp[1] += disp[0];
    disp[0] = 0.f;
}

}  // namespace crk

using namespace crk;

static unsigned nb256(int64_t n) { return (unsigned)((n + 255) / 256); }

extern "C" {

crk_status crk_courant_dt(crk_ctx* c, crk_particles* p, float c_cfl, float c_acc, float* dt_out, void* stream) {
    if (!c || !p || !dt_out || !(c_cfl > 0.f) || !(c_acc > 0.f)) return c ? fail(c, CRK_EINVAL, "bad args") : CRK_EINVAL;
    if (c->stage < ST_EXT) return fail(c, CRK_ESTATE, "call crk_hydro_accel_dudt first (needs c and a_h)");
    if (!p->ax || !p->ay || !p->az || !p->ahx || !p->ahy || !p->ahz || !p->H || !p->species)
        return fail(c, CRK_EINVAL, "courant needs a, a_h, H, species");
    cudaStream_t st = (cudaStream_t)stream;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_set_inf<<<1, 1, 0, st>>>(dt_out);
    CRK_LAUNCHED(c, "courant init");
    const int64_t n = p->n;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    const int64_t grid = std::min<int64_t>(nb256(n), (int64_t)nsm * 8);
    k_courant<<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, st>>>(
        n, p->species, P<int32_t>(c->grank), P<float4>(c->grec), p->H, p->ax, p->ay, p->az, p->ahx, p->ahy, p->ahz,
        sqrtf(c->prm.eps2), c_cfl, c_acc, dt_out);
    CRK_LAUNCHED(c, "courant");
    return CRK_OK;
}

crk_status crk_kick(crk_ctx* c, crk_particles* p, float dt, void* stream) {
    if (!c || !p) return CRK_EINVAL;
    if (!p->ax || !p->ay || !p->az || !p->ahx || !p->ahy || !p->ahz || !p->dudt || !p->vx || !p->vy || !p->vz ||
        !p->u || !p->species)
        return fail(c, CRK_EINVAL, "kick needs a, a_h, du/dt, v, u, species");
    if (p->n <= 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_kick<<<nb256(p->n), 256, 0, (cudaStream_t)stream>>>(p->n, p->species, dt, p->ax, p->ay, p->az, p->ahx, p->ahy,
                                                         p->ahz, p->dudt, p->vx, p->vy, p->vz, p->u);
    CRK_LAUNCHED(c, "kick");
    return CRK_OK;
}

crk_status crk_drift(crk_ctx* c, crk_particles* p, float dt, void* stream) {
    if (!c || !p) return CRK_EINVAL;
    if (!p->x || !p->y || !p->z || !p->vx || !p->vy || !p->vz) return fail(c, CRK_EINVAL, "drift needs x, v");
    if (p->n <= 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    const bool skin = c->skin_lists && p->n == c->n;  // keep the skin lists: no wrap, track the displacement
    k_drift<<<nb256(p->n), 256, 0, (cudaStream_t)stream>>>(p->n, dt, c->lay.inv_q, (float)c->lay.q, c->lay.L[0],
                                                          c->lay.L[1], c->lay.L[2], p->x, p->y, p->z, p->vx, p->vy,
                                                          p->vz, !skin, skin ? P<float>(c->disp) : nullptr);
    CRK_LAUNCHED(c, "drift");
    if (skin) {
        k_disp_accum<<<1, 1, 0, (cudaStream_t)stream>>>(P<float>(c->disp));
        CRK_LAUNCHED(c, "displacement bound");
    }
    c->stage = ST_NONE;  // positions moved: crk_build_lists (or crk_refresh with a skin) before the next pass
    return CRK_OK;
}

crk_status crk_refresh(crk_ctx* c, crk_particles* p, void* stream) {
    if (!c || !p) return CRK_EINVAL;
    if (!p->x || !p->y || !p->z || !p->m || !p->H || p->n != c->n) return fail(c, CRK_EINVAL, "refresh needs x, m, H");
    if (!c->skin_lists) return fail(c, CRK_ESTATE, "no skin lists to refresh: call crk_build_lists");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    return refresh(c, p, (cudaStream_t)stream);
}

}  // extern "C"
