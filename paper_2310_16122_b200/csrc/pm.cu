// pm.cu — long-range gravity by particle-mesh (the force split of
// long-range particle-mesh + short-range direct particle-particle).
// One GPU: cloud-in-cell deposit of the mass, forward real-to-complex FFT (cuFFT), the
// Gaussian-filtered Poisson kernel -4 pi G exp(-k^2 r_s^2) / k^2 with a spectral gradient
// (-i k), three inverse FFTs and cloud-in-cell interpolation of the acceleration.  The filter
// makes the long-range force of a point mass G m / r^2 [erf(r / 2 r_s) - (r / (r_s sqrt(pi)))
// exp(-r^2 / 4 r_s^2)], the counterpart of the short-range force whose grid polynomial
// gen/configs.py fits (O5).  Readings in DESIGN.md §2 ("Long-range PM").
#include <cufft.h>

#include <cmath>
#include <new>

#include "common.cuh"

struct crk_pm {
    int ng = 0;
    float L = 0.f, rs = 0.f, G = 0.f;
    int device = 0;
    cufftHandle fwd = 0, inv = 0;
    float* rho = nullptr;          // ng^3 real
    cufftComplex* rk = nullptr;    // ng^2 (ng/2 + 1)
    cufftComplex* ak[3] = {nullptr, nullptr, nullptr};
    float* ag[3] = {nullptr, nullptr, nullptr};
    // slab decomposition (crk_pm_slab_create): rank owns x-planes [rank nxl, (rank+1) nxl) of the
    // real mesh and y-rows [rank nyl, (rank+1) nyl) of the half-complex spectrum
    bool slab = false;
    int rank = 0, P = 1, nxl = 0, nyl = 0, nzc = 0;
    cufftHandle f2 = 0, i2 = 0, f1 = 0, i1 = 0;
    cufftComplex* c2 = nullptr;  // 3 nxl ng nzc: 2-D spectra of the owned planes
    cufftComplex* t1 = nullptr;  // 3 nyl nzc ng: owned spectrum rows, x contiguous
};

namespace crk {

// CIC weights of coordinate x (grid units, periodic): cells i0, i0 + 1 with weights 1 - f, f
__device__ __forceinline__ void cic1(float x, int ng, int& i0, int& i1, float& w0, float& w1) {
    const float s = x - 0.5f;  // cell centres at (i + 1/2)
    const float fl = floorf(s);
    const float f = s - fl;
    int i = (int)fl;
    i0 = ((i % ng) + ng) % ng;
    i1 = (i0 + 1) % ng;
    w0 = 1.f - f;
    w1 = f;
}

__global__ void k_cic_deposit(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                              const float* __restrict__ z, const float* __restrict__ m, float inv_dx, int ng,
                              float inv_cell_vol, float* rho) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int ix[2], iy[2], iz[2];
    float wx[2], wy[2], wz[2];
    cic1(x[p] * inv_dx, ng, ix[0], ix[1], wx[0], wx[1]);
    cic1(y[p] * inv_dx, ng, iy[0], iy[1], wy[0], wy[1]);
    cic1(z[p] * inv_dx, ng, iz[0], iz[1], wz[0], wz[1]);
    const float mm = m[p] * inv_cell_vol;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                atomicAdd(rho + ((int64_t)ix[a] * ng + iy[b]) * ng + iz[c], mm * wx[a] * wy[b] * wz[c]);
}

// a_k = -i k phi_k, phi_k = -4 pi G exp(-k^2 rs^2) / k^2 rho_k / ng^3 (inverse FFT unnormalised);
// the Nyquist component of each derivative is zeroed (an odd operator there is ill-defined)
__global__ void k_green(int ng, float L, float rs, float G, const cufftComplex* __restrict__ rk, cufftComplex* ax,
                        cufftComplex* ay, cufftComplex* az) {
    const int nz = ng / 2 + 1;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)ng * ng * nz) return;
    const int k = (int)(t % nz), j = (int)((t / nz) % ng), i = (int)(t / ((int64_t)nz * ng));
    const float w = 6.283185307179586f / L;
    const int si = i <= ng / 2 ? i : i - ng, sj = j <= ng / 2 ? j : j - ng;
    const float kx = w * si, ky = w * sj, kz = w * k;
    const float k2 = kx * kx + ky * ky + kz * kz;
    float g = 0.f;
    if (k2 > 0.f) g = -12.566370614359172f * G * expf(-k2 * rs * rs) / (k2 * (float)ng * (float)ng * (float)ng);
    const cufftComplex r = rk[t];
    const float pr = g * r.x, pi = g * r.y;  // phi_k
    // -i k phi = (k pi, -k pr)
    const float dx = (i == ng / 2) ? 0.f : kx, dy = (j == ng / 2) ? 0.f : ky, dz = (k == ng / 2) ? 0.f : kz;
    ax[t] = make_cuComplex(dx * pi, -dx * pr);
    ay[t] = make_cuComplex(dy * pi, -dy * pr);
    az[t] = make_cuComplex(dz * pi, -dz * pr);
}

__global__ void k_cic_interp(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                             const float* __restrict__ z, float inv_dx, int ng, const float* __restrict__ gx,
                             const float* __restrict__ gy, const float* __restrict__ gz, float* ax, float* ay,
                             float* az) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int ix[2], iy[2], iz[2];
    float wx[2], wy[2], wz[2];
    cic1(x[p] * inv_dx, ng, ix[0], ix[1], wx[0], wx[1]);
    cic1(y[p] * inv_dx, ng, iy[0], iy[1], wy[0], wy[1]);
    cic1(z[p] * inv_dx, ng, iz[0], iz[1], wz[0], wz[1]);
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int64_t q = ((int64_t)ix[a] * ng + iy[b]) * ng + iz[c];
                const float w = wx[a] * wy[b] * wz[c];
                sx = fmaf(w, gx[q], sx);
                sy = fmaf(w, gy[q], sy);
                sz = fmaf(w, gz[q], sz);
            }
    ax[p] = sx;
    ay[p] = sy;
    az[p] = sz;
}

// ---- slab decomposition: pack / unpack between the plane layout [ixl][iy][kz] and the
// pencil layout [iyl][kz][X] (X contiguous for the 1-D transforms along x) ----

// C[ixl][iy][kz] -> send[r'][ixl][iyl][kz], r' = iy / nyl
__global__ void k_slab_pack_fwd(int nxl, int ng, int nyl, int nzc, const cufftComplex* __restrict__ c,
                                cufftComplex* send) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nxl * ng * nzc) return;
    const int kz = (int)(t % nzc), iy = (int)((t / nzc) % ng), ixl = (int)(t / ((int64_t)nzc * ng));
    const int r = iy / nyl, iyl = iy % nyl;
    send[(((int64_t)r * nxl + ixl) * nyl + iyl) * nzc + kz] = c[t];
}

// recv[r''][ixl][iyl][kz] (x range of rank r'') -> T[iyl][kz][X], X = r'' nxl + ixl
__global__ void k_slab_unpack_x(int nxl, int ng, int nyl, int nzc, const cufftComplex* __restrict__ recv,
                                cufftComplex* t1) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)ng * nyl * nzc) return;
    const int kz = (int)(t % nzc), iyl = (int)((t / nzc) % nyl), X = (int)(t / ((int64_t)nzc * nyl));
    const int r = X / nxl, ixl = X % nxl;
    t1[((int64_t)iyl * nzc + kz) * ng + X] = recv[(((int64_t)r * nxl + ixl) * nyl + iyl) * nzc + kz];
}

// the Green's function and spectral gradient of k_green on the pencil layout:
// T[iyl][kz][X] -> T3[c][iyl][kz][X]
__global__ void k_green_pencil(int ng, int nyl, int nzc, int y0, float L, float rs, float G,
                               const cufftComplex* __restrict__ t1, cufftComplex* t3) {
    const int64_t nt = (int64_t)nyl * nzc * ng;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int i = (int)(t % ng), k = (int)((t / ng) % nzc), j = y0 + (int)(t / ((int64_t)ng * nzc));
    const float w = 6.283185307179586f / L;
    const int si = i <= ng / 2 ? i : i - ng, sj = j <= ng / 2 ? j : j - ng;
    const float kx = w * si, ky = w * sj, kz = w * k;
    const float k2 = kx * kx + ky * ky + kz * kz;
    float g = 0.f;
    if (k2 > 0.f) g = -12.566370614359172f * G * expf(-k2 * rs * rs) / (k2 * (float)ng * (float)ng * (float)ng);
    const cufftComplex r = t1[t];
    const float pr = g * r.x, pi = g * r.y;
    const float dx = (i == ng / 2) ? 0.f : kx, dy = (j == ng / 2) ? 0.f : ky, dz = (k == ng / 2) ? 0.f : kz;
    t3[t] = make_cuComplex(dx * pi, -dx * pr);
    t3[nt + t] = make_cuComplex(dy * pi, -dy * pr);
    t3[2 * nt + t] = make_cuComplex(dz * pi, -dz * pr);
}

// T3[c][iyl][kz][X] -> send3[r''][c][ixl][iyl][kz], r'' = X / nxl
__global__ void k_slab_pack_back(int nxl, int ng, int nyl, int nzc, const cufftComplex* __restrict__ t3,
                                 cufftComplex* send) {
    const int64_t nt = (int64_t)nyl * nzc * ng;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= 3 * nt) return;
    const int c = (int)(t / nt);
    const int64_t u = t % nt;
    const int kz = (int)(u % nzc), iyl = (int)((u / nzc) % nyl), X = (int)(u / ((int64_t)nzc * nyl));
    const int r = X / nxl, ixl = X % nxl;
    send[((((int64_t)r * 3 + c) * nxl + ixl) * nyl + iyl) * nzc + kz] =
        t3[(int64_t)c * nt + ((int64_t)iyl * nzc + kz) * ng + X];
}

// recv3[r][c][ixl][iyl][kz] (y range of rank r) -> C3[c][ixl][iy][kz], iy = r nyl + iyl
__global__ void k_slab_unpack_back(int nxl, int ng, int nyl, int nzc, const cufftComplex* __restrict__ recv,
                                   cufftComplex* c3) {
    const int64_t n1 = (int64_t)nxl * ng * nzc;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= 3 * n1) return;
    const int c = (int)(t / n1);
    const int64_t u = t % n1;
    const int kz = (int)(u % nzc), iy = (int)((u / nzc) % ng), ixl = (int)(u / ((int64_t)nzc * ng));
    const int r = iy / nyl, iyl = iy % nyl;
    c3[t] = recv[((((int64_t)r * 3 + c) * nxl + ixl) * nyl + iyl) * nzc + kz];
}

// CIC interpolation from the gathered slabs acc[r][c][ixl][iy][iz] (X = r nxl + ixl)
__global__ void k_cic_interp_slabs(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                                   const float* __restrict__ z, float inv_dx, int ng, int nxl,
                                   const float* __restrict__ acc, float* ax, float* ay, float* az) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int ix[2], iy[2], iz[2];
    float wx[2], wy[2], wz[2];
    cic1(x[p] * inv_dx, ng, ix[0], ix[1], wx[0], wx[1]);
    cic1(y[p] * inv_dx, ng, iy[0], iy[1], wy[0], wy[1]);
    cic1(z[p] * inv_dx, ng, iz[0], iz[1], wz[0], wz[1]);
    const int64_t plane = (int64_t)ng * ng;
    float s[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const int r = ix[a] / nxl, xl = ix[a] % nxl;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float* g = acc + ((int64_t)(r * 3 + c) * nxl + xl) * plane;
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int d = 0; d < 2; ++d) s[c] = fmaf(wx[a] * wy[b] * wz[d], g[(int64_t)iy[b] * ng + iz[d]], s[c]);
        }
    }
    ax[p] = s[0];
    ay[p] = s[1];
    az[p] = s[2];
}

}  // namespace crk

using namespace crk;

static unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

extern "C" {

crk_status crk_pm_create(int n_grid, const double* box, float r_s, float G, int device, crk_pm** out) {
    if (!out || !box) return CRK_EINVAL;
    *out = nullptr;
    if (n_grid < 8 || n_grid > 1024 || (n_grid & (n_grid - 1)) || !(r_s > 0.f)) return CRK_EINVAL;
    if (!(box[0] > 0.0) || box[1] != box[0] || box[2] != box[0]) return CRK_EINVAL;  // cubic boxes
    if (cudaSetDevice(device) != cudaSuccess) return CRK_ECUDA;
    crk_pm* pm = new (std::nothrow) crk_pm();
    if (!pm) return CRK_ENOMEM;
    pm->ng = n_grid;
    pm->L = (float)box[0];
    pm->rs = r_s;
    pm->G = G;
    pm->device = device;
    const size_t nr = (size_t)n_grid * n_grid * n_grid, nc = (size_t)n_grid * n_grid * (n_grid / 2 + 1);
    bool ok = cudaMalloc(&pm->rho, nr * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&pm->rk, nc * sizeof(cufftComplex)) == cudaSuccess;
    for (int a = 0; a < 3 && ok; ++a)
        ok = cudaMalloc(&pm->ak[a], nc * sizeof(cufftComplex)) == cudaSuccess &&
             cudaMalloc(&pm->ag[a], nr * sizeof(float)) == cudaSuccess;
    ok = ok && cufftPlan3d(&pm->fwd, n_grid, n_grid, n_grid, CUFFT_R2C) == CUFFT_SUCCESS &&
         cufftPlan3d(&pm->inv, n_grid, n_grid, n_grid, CUFFT_C2R) == CUFFT_SUCCESS;
    if (!ok) {
        crk_pm_destroy(pm);
        return CRK_ENOMEM;
    }
    *out = pm;
    return CRK_OK;
}

crk_status crk_pm_destroy(crk_pm* pm) {
    if (!pm) return CRK_EINVAL;
    cudaSetDevice(pm->device);
    cudaDeviceSynchronize();
    if (pm->fwd) cufftDestroy(pm->fwd);
    if (pm->inv) cufftDestroy(pm->inv);
    for (cufftHandle h : {pm->f2, pm->i2, pm->f1, pm->i1})
        if (h) cufftDestroy(h);
    cudaFree(pm->c2);
    cudaFree(pm->t1);
    cudaFree(pm->rho);
    cudaFree(pm->rk);
    for (int a = 0; a < 3; ++a) {
        cudaFree(pm->ak[a]);
        cudaFree(pm->ag[a]);
    }
    delete pm;
    return CRK_OK;
}

crk_status crk_pm_slab_create(int n_grid, const double* box, float r_s, float G, int rank, int nranks,
                              int device, crk_pm** out) {
    if (!out || !box) return CRK_EINVAL;
    *out = nullptr;
    if (n_grid < 8 || n_grid > 1024 || (n_grid & (n_grid - 1)) || !(r_s > 0.f)) return CRK_EINVAL;
    if (!(box[0] > 0.0) || box[1] != box[0] || box[2] != box[0]) return CRK_EINVAL;
    if (nranks < 1 || n_grid % nranks || rank < 0 || rank >= nranks) return CRK_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return CRK_ECUDA;
    crk_pm* pm = new (std::nothrow) crk_pm();
    if (!pm) return CRK_ENOMEM;
    pm->ng = n_grid;
    pm->L = (float)box[0];
    pm->rs = r_s;
    pm->G = G;
    pm->device = device;
    pm->slab = true;
    pm->rank = rank;
    pm->P = nranks;
    pm->nxl = n_grid / nranks;
    pm->nyl = n_grid / nranks;
    pm->nzc = n_grid / 2 + 1;
    const int ng = n_grid, nxl = pm->nxl, nyl = pm->nyl, nzc = pm->nzc;
    int n2[2] = {ng, ng};
    bool ok = cudaMalloc(&pm->c2, 3 * (size_t)nxl * ng * nzc * sizeof(cufftComplex)) == cudaSuccess &&
              cudaMalloc(&pm->t1, 4 * (size_t)nyl * nzc * ng * sizeof(cufftComplex)) == cudaSuccess;
    ok = ok && cufftPlanMany(&pm->f2, 2, n2, nullptr, 1, 0, nullptr, 1, 0, CUFFT_R2C, nxl) == CUFFT_SUCCESS &&
         cufftPlanMany(&pm->i2, 2, n2, nullptr, 1, 0, nullptr, 1, 0, CUFFT_C2R, 3 * nxl) == CUFFT_SUCCESS &&
         cufftPlan1d(&pm->f1, ng, CUFFT_C2C, nyl * nzc) == CUFFT_SUCCESS &&
         cufftPlan1d(&pm->i1, ng, CUFFT_C2C, 3 * nyl * nzc) == CUFFT_SUCCESS;
    if (!ok) {
        crk_pm_destroy(pm);
        return CRK_ENOMEM;
    }
    *out = pm;
    return CRK_OK;
}

crk_status crk_pm_deposit(crk_pm* pm, int64_t n, const float* x, const float* y, const float* z, const float* m,
                          float* rho_full, void* stream) {
    if (!pm || !rho_full || n < 0 || (n > 0 && (!x || !y || !z || !m))) return CRK_EINVAL;
    if (cudaSetDevice(pm->device) != cudaSuccess) return CRK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int ng = pm->ng;
    const float dx = pm->L / ng;
    if (zero_async(rho_full, (size_t)ng * ng * ng * sizeof(float), st) != cudaSuccess) return CRK_ECUDA;
    if (n > 0) k_cic_deposit<<<nb(n), 256, 0, st>>>(n, x, y, z, m, 1.f / dx, ng, 1.f / (dx * dx * dx), rho_full);
    return cudaGetLastError() == cudaSuccess ? CRK_OK : CRK_ECUDA;
}

crk_status crk_pm_slab_forward(crk_pm* pm, const float* rho_slab, void* send, void* stream) {
    if (!pm || !pm->slab || !rho_slab || !send) return CRK_EINVAL;
    if (cudaSetDevice(pm->device) != cudaSuccess) return CRK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    if (cufftSetStream(pm->f2, st) != CUFFT_SUCCESS ||
        cufftExecR2C(pm->f2, const_cast<float*>(rho_slab), pm->c2) != CUFFT_SUCCESS)
        return CRK_ECUDA;
    const int64_t nc = (int64_t)pm->nxl * pm->ng * pm->nzc;
    k_slab_pack_fwd<<<nb(nc), 256, 0, st>>>(pm->nxl, pm->ng, pm->nyl, pm->nzc, pm->c2, (cufftComplex*)send);
    return cudaGetLastError() == cudaSuccess ? CRK_OK : CRK_ECUDA;
}

crk_status crk_pm_slab_solve(crk_pm* pm, const void* recv, void* send3, void* stream) {
    if (!pm || !pm->slab || !recv || !send3) return CRK_EINVAL;
    if (cudaSetDevice(pm->device) != cudaSuccess) return CRK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int ng = pm->ng, nyl = pm->nyl, nzc = pm->nzc;
    const int64_t nt = (int64_t)nyl * nzc * ng;
    cufftComplex* t1 = pm->t1;
    cufftComplex* t3 = pm->t1 + nt;
    k_slab_unpack_x<<<nb(nt), 256, 0, st>>>(pm->nxl, ng, nyl, nzc, (const cufftComplex*)recv, t1);
    if (cufftSetStream(pm->f1, st) != CUFFT_SUCCESS || cufftSetStream(pm->i1, st) != CUFFT_SUCCESS ||
        cufftExecC2C(pm->f1, t1, t1, CUFFT_FORWARD) != CUFFT_SUCCESS)
        return CRK_ECUDA;
    k_green_pencil<<<nb(nt), 256, 0, st>>>(ng, nyl, nzc, pm->rank * nyl, pm->L, pm->rs, pm->G, t1, t3);
    if (cufftExecC2C(pm->i1, t3, t3, CUFFT_INVERSE) != CUFFT_SUCCESS) return CRK_ECUDA;
    k_slab_pack_back<<<nb(3 * nt), 256, 0, st>>>(pm->nxl, ng, nyl, nzc, t3, (cufftComplex*)send3);
    return cudaGetLastError() == cudaSuccess ? CRK_OK : CRK_ECUDA;
}

crk_status crk_pm_slab_inverse(crk_pm* pm, const void* recv3, float* acc_slab, void* stream) {
    if (!pm || !pm->slab || !recv3 || !acc_slab) return CRK_EINVAL;
    if (cudaSetDevice(pm->device) != cudaSuccess) return CRK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n1 = (int64_t)pm->nxl * pm->ng * pm->nzc;
    k_slab_unpack_back<<<nb(3 * n1), 256, 0, st>>>(pm->nxl, pm->ng, pm->nyl, pm->nzc,
                                                    (const cufftComplex*)recv3, pm->c2);
    if (cufftSetStream(pm->i2, st) != CUFFT_SUCCESS || cufftExecC2R(pm->i2, pm->c2, acc_slab) != CUFFT_SUCCESS)
        return CRK_ECUDA;
    return cudaGetLastError() == cudaSuccess ? CRK_OK : CRK_ECUDA;
}

crk_status crk_pm_interp(crk_pm* pm, int64_t n, const float* x, const float* y, const float* z,
                         const float* acc_full, float* ax, float* ay, float* az, void* stream) {
    if (!pm || !pm->slab || !acc_full || n < 0 || (n > 0 && (!x || !y || !z || !ax || !ay || !az)))
        return CRK_EINVAL;
    if (cudaSetDevice(pm->device) != cudaSuccess) return CRK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const float dx = pm->L / pm->ng;
    if (n > 0)
        k_cic_interp_slabs<<<nb(n), 256, 0, st>>>(n, x, y, z, 1.f / dx, pm->ng, pm->nxl, acc_full, ax, ay, az);
    return cudaGetLastError() == cudaSuccess ? CRK_OK : CRK_ECUDA;
}

crk_status crk_pm_accel(crk_pm* pm, int64_t n, const float* x, const float* y, const float* z, const float* m,
                        float* ax, float* ay, float* az, void* stream) {
    if (!pm || pm->slab || n < 0 || (n > 0 && (!x || !y || !z || !m || !ax || !ay || !az))) return CRK_EINVAL;
    if (cudaSetDevice(pm->device) != cudaSuccess) return CRK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int ng = pm->ng;
    const size_t nr = (size_t)ng * ng * ng, nc = (size_t)ng * ng * (ng / 2 + 1);
    const float dx = pm->L / ng;
    if (zero_async(pm->rho, nr * sizeof(float), st) != cudaSuccess) return CRK_ECUDA;
    if (n > 0) k_cic_deposit<<<nb(n), 256, 0, st>>>(n, x, y, z, m, 1.f / dx, ng, 1.f / (dx * dx * dx), pm->rho);
    if (cufftSetStream(pm->fwd, st) != CUFFT_SUCCESS || cufftSetStream(pm->inv, st) != CUFFT_SUCCESS ||
        cufftExecR2C(pm->fwd, pm->rho, pm->rk) != CUFFT_SUCCESS)
        return CRK_ECUDA;
    k_green<<<nb((int64_t)nc), 256, 0, st>>>(ng, pm->L, pm->rs, pm->G, pm->rk, pm->ak[0], pm->ak[1], pm->ak[2]);
    for (int a = 0; a < 3; ++a)
        if (cufftExecC2R(pm->inv, pm->ak[a], pm->ag[a]) != CUFFT_SUCCESS) return CRK_ECUDA;
    if (n > 0)
        k_cic_interp<<<nb(n), 256, 0, st>>>(n, x, y, z, 1.f / dx, ng, pm->ag[0], pm->ag[1], pm->ag[2], ax, ay, az);
    return cudaGetLastError() == cudaSuccess ? CRK_OK : CRK_ECUDA;
}

}  // extern "C"
