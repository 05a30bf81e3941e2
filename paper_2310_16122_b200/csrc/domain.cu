// domain.cu — a9: ghost-exchange support for the 3-D domain decomposition
// (SURVEY.md §8(a) a9, §8(e)).  Leaf-granular (whole chaining-mesh cells) selection of
// the particles / gas ranks a peer needs, and packing of the three exchange rounds:
// R1 whole particles before the sort, R2 the volume V after Geometry, R3 the accel
// record after Extras.  The transfers themselves are NCCL send/recv (torch.distributed)
// issued by the caller; these kernels only gather and scatter.
#include <cub/cub.cuh>

#include "common.cuh"

namespace crk {

__global__ void k_cell_flags(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                             const float* __restrict__ z, const uint8_t* __restrict__ sp, int gas_only, float inv_q,
                             int cs, const uint8_t* __restrict__ mx, const uint8_t* __restrict__ my,
                             const uint8_t* __restrict__ mz, uint8_t* flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t cx = (uint32_t)(x[i] * inv_q) >> cs, cy = (uint32_t)(y[i] * inv_q) >> cs,
                   cz = (uint32_t)(z[i] * inv_q) >> cs;
    bool f = mx[cx] && my[cy] && mz[cz];
    if (gas_only && sp) f = f && sp[i] == 1;
    flag[i] = f ? 1 : 0;
}

__global__ void k_cell_flags_gas(int64_t ng, const float4* __restrict__ gpos, float inv_q, int cs,
                                 const uint8_t* __restrict__ mx, const uint8_t* __restrict__ my,
                                 const uint8_t* __restrict__ mz, uint8_t* flag) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ng) return;
    const float4 p = gpos[k];
    const uint32_t cx = (uint32_t)(p.x * inv_q) >> cs, cy = (uint32_t)(p.y * inv_q) >> cs,
                   cz = (uint32_t)(p.z * inv_q) >> cs;
    flag[k] = (mx[cx] && my[cy] && mz[cz]) ? 1 : 0;
}

struct Rec48 {
    float f[9];
    float sp;
    int64_t id;
};
static_assert(sizeof(Rec48) == 48, "packed particle record");

__global__ void k_pack_particles(int64_t n, const int32_t* __restrict__ idx, const float* x, const float* y,
                                 const float* z, const float* vx, const float* vy, const float* vz, const float* m,
                                 const float* H, const float* u, const uint8_t* sp, const int64_t* id, Rec48* out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t i = idx[t];
    Rec48 r;
    r.f[0] = x[i]; r.f[1] = y[i]; r.f[2] = z[i];
    r.f[3] = vx[i]; r.f[4] = vy[i]; r.f[5] = vz[i];
    r.f[6] = m[i]; r.f[7] = H[i]; r.f[8] = u[i];
    r.sp = (float)sp[i];
    r.id = id[i];
    out[t] = r;
}

__global__ void k_unpack_particles(int64_t n, int64_t off, const Rec48* __restrict__ in, float* x, float* y, float* z,
                                   float* vx, float* vy, float* vz, float* m, float* H, float* u, uint8_t* sp,
                                   int64_t* id) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const Rec48 r = in[t];
    const int64_t i = off + t;
    x[i] = r.f[0]; y[i] = r.f[1]; z[i] = r.f[2];
    vx[i] = r.f[3]; vy[i] = r.f[4]; vz[i] = r.f[5];
    m[i] = r.f[6]; H[i] = r.f[7]; u[i] = r.f[8];
    sp[i] = (uint8_t)r.sp;
    id[i] = r.id;
}

// accel record of gas rank k, component c < 9 (hydro.cu load_rec)
__device__ __forceinline__ int64_t rec_at(int64_t ng, int64_t k, int c) { return (void)ng, 9 * k + c; }

__global__ void k_pack_gas(int64_t n, int what, const int32_t* __restrict__ idx, const float* __restrict__ gV,
                           const float4* __restrict__ grec, int64_t ng, void* out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (what == 0) {
        if (t < n) reinterpret_cast<float*>(out)[t] = gV[idx[t]];
    } else {
        if (t >= n * 9) return;
        const int64_t k = t / 9;
        reinterpret_cast<float4*>(out)[t] = grec[rec_at(ng, idx[k], (int)(t % 9))];
    }
}

__global__ void k_unpack_gas(int64_t n, int what, const int32_t* __restrict__ idx, const void* in,
                             const float4* __restrict__ gpos, float* gV, float4* gposV, float4* grec, int64_t ng) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (what == 0) {
        if (t >= n) return;
        const float V = reinterpret_cast<const float*>(in)[t];
        const int32_t k = idx[t];
        const float4 p = gpos[k];  // ghost rows of the corrections/extras j-tiles: (x, y, z, V)
        gV[k] = V;
        gposV[k] = make_float4(p.x, p.y, p.z, V);
    } else {
        if (t >= n * 9) return;
        const int64_t k = t / 9;
        grec[rec_at(ng, idx[k], (int)(t % 9))] = reinterpret_cast<const float4*>(in)[t];
    }
}

// records [0, min(*count, cap)) of a selection whose size is a device scalar (no host sync)
__global__ void k_pack_particles_dev(int64_t cap, const int32_t* __restrict__ count, const int32_t* __restrict__ idx,
                                     const float* x, const float* y, const float* z, const float* vx,
                                     const float* vy, const float* vz, const float* m, const float* H, const float* u,
                                     const uint8_t* sp, const int64_t* id, Rec48* out) {
    const int64_t n = min((int64_t)*count, cap);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[t];
        Rec48 r;
        r.f[0] = x[i]; r.f[1] = y[i]; r.f[2] = z[i];
        r.f[3] = vx[i]; r.f[4] = vy[i]; r.f[5] = vz[i];
        r.f[6] = m[i]; r.f[7] = H[i]; r.f[8] = u[i];
        r.sp = (float)sp[i];
        r.id = id[i];
        out[t] = r;
    }
}

// R2 with velocities: (V, vx, vy, vz) of gas rank idx[t] — the volume and the gravity-kicked
// velocity the owner's Extras sees (the ghost copy from R1 predates the owner's kick)
__global__ void k_pack_gas_state(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ gas_idx,
                                 const float* __restrict__ gV, const float* vx, const float* vy, const float* vz,
                                 float4* out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int32_t k = idx[t];
    const int64_t i = gas_idx[k];
    out[t] = make_float4(gV[k], vx[i], vy[i], vz[i]);
}

__global__ void k_unpack_gas_state(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ gas_idx,
                                   const float4* __restrict__ in, const float4* __restrict__ gpos, float* gV,
                                   float4* gposV, float* vx, float* vy, float* vz) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const float4 r = in[t];
    const int32_t k = idx[t];
    const int64_t i = gas_idx[k];
    const float4 p = gpos[k];
    gV[k] = r.x;
    gposV[k] = make_float4(p.x, p.y, p.z, r.x);
    vx[i] = r.y; vy[i] = r.z; vz[i] = r.w;
}

static inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

static crk_status upload_masks(crk_ctx* c, const uint8_t* mx, const uint8_t* my, const uint8_t* mz,
                               cudaStream_t st, uint8_t** d) {
    const int* nc = c->lay.ncell;
    CRK_TRY(grow(c, c->sel_mask, (size_t)(nc[0] + nc[1] + nc[2]), st));
    uint8_t* base = P<uint8_t>(c->sel_mask);
    const uint8_t* src[3] = {mx, my, mz};
    int64_t o = 0;
    for (int a = 0; a < 3; ++a) {
        if (!src[a]) return fail(c, CRK_EINVAL, "null cell mask");
        CRK_TRY(cuda_check(c, cudaMemcpyAsync(base + o, src[a], nc[a], cudaMemcpyHostToDevice, st), "mask h2d"));
        d[a] = base + o;
        o += nc[a];
    }
    return CRK_OK;
}

static crk_status compact(crk_ctx* c, int64_t n, int32_t* idx_out, int64_t* count_out, cudaStream_t st) {
    CRK_TRY(grow(c, c->dev_scalars, 64, st));
    size_t tmp = 0;
    int64_t* dnum = reinterpret_cast<int64_t*>(P<char>(c->dev_scalars) + 32);
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, tmp, it, P<uint8_t>(c->sel_flag), idx_out, dnum, (int)n, st);
    CRK_TRY(grow(c, c->cub_tmp, tmp, st));
    tmp = c->cub_tmp.cap;
    CRK_TRY(cuda_check(c, cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, it, P<uint8_t>(c->sel_flag), idx_out, dnum,
                                                     (int)n, st), "select"));
    c->launches += 2;
    volatile int64_t* host = reinterpret_cast<int64_t*>(P<char>(c->pinned) + 128);
    Readback rb;
    rb.add(dnum, 128, 8);
    CRK_TRY(readback(c, rb, st));
    CRK_TRY(cuda_check(c, cudaStreamSynchronize(st), "sync"));
    *count_out = *host;
    return CRK_OK;
}

// device-count variant: the number selected goes to *count_dev (int32), no host sync
static crk_status compact_dev(crk_ctx* c, int64_t n, int32_t* idx_out, int32_t* count_dev, cudaStream_t st) {
    size_t tmp = 0;
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, tmp, it, P<uint8_t>(c->sel_flag), idx_out, count_dev, (int)n, st);
    CRK_TRY(grow(c, c->cub_tmp, tmp, st));
    tmp = c->cub_tmp.cap;
    CRK_TRY(cuda_check(c, cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, it, P<uint8_t>(c->sel_flag), idx_out,
                                                     count_dev, (int)n, st), "select"));
    c->launches += 2;
    return CRK_OK;
}

}  // namespace crk

using namespace crk;

extern "C" {

crk_status crk_select_cells(crk_ctx* c, const float* x, const float* y, const float* z, const uint8_t* species,
                            int gas_only, int64_t n, const uint8_t* mask_x, const uint8_t* mask_y,
                            const uint8_t* mask_z, int32_t* idx_out, int64_t* count_out, void* stream) {
    if (!c || !count_out || n < 0 || (n > 0 && (!x || !y || !z || !idx_out))) return fail(c, CRK_EINVAL, "bad args");
    if (gas_only && !species) return fail(c, CRK_EINVAL, "gas_only needs species");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    *count_out = 0;
    if (n == 0) return CRK_OK;
    uint8_t* dm[3];
    CRK_TRY(upload_masks(c, mask_x, mask_y, mask_z, st, dm));
    CRK_TRY(grow(c, c->sel_flag, n, st));
    k_cell_flags<<<nb(n), 256, 0, st>>>(n, x, y, z, species, gas_only, c->lay.inv_q, c->lay.cs, dm[0], dm[1], dm[2],
                                        P<uint8_t>(c->sel_flag));
    CRK_LAUNCHED(c, "cell flags");
    return compact(c, n, idx_out, count_out, st);
}

crk_status crk_select_gas(crk_ctx* c, const uint8_t* mask_x, const uint8_t* mask_y, const uint8_t* mask_z,
                          int32_t* idx_out, int64_t* count_out, void* stream) {
    if (!c || !count_out) return CRK_EINVAL;
    if (c->stage < ST_LISTS) return fail(c, CRK_ESTATE, "call crk_build_lists first");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    *count_out = 0;
    const int64_t ng = c->n_gas;
    if (ng == 0) return CRK_OK;
    if (!idx_out) return fail(c, CRK_EINVAL, "null idx_out");
    uint8_t* dm[3];
    CRK_TRY(upload_masks(c, mask_x, mask_y, mask_z, st, dm));
    CRK_TRY(grow(c, c->sel_flag, ng, st));
    k_cell_flags_gas<<<nb(ng), 256, 0, st>>>(ng, P<float4>(c->gpos), c->lay.inv_q, c->lay.cs, dm[0], dm[1], dm[2],
                                             P<uint8_t>(c->sel_flag));
    CRK_LAUNCHED(c, "gas cell flags");
    return compact(c, ng, idx_out, count_out, st);
}

crk_status crk_select_cells_dev(crk_ctx* c, const float* x, const float* y, const float* z, const uint8_t* species,
                                int gas_only, int64_t n, const uint8_t* dmask, int32_t* idx_out, int32_t* count_dev,
                                void* stream) {
    if (!c || !count_dev || !dmask || n < 0 || (n > 0 && (!x || !y || !z || !idx_out)))
        return fail(c, CRK_EINVAL, "bad args");
    if (gas_only && !species) return fail(c, CRK_EINVAL, "gas_only needs species");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return cuda_check(c, zero_async(count_dev, 4, st, c), "memset");
    CRK_TRY(grow(c, c->sel_flag, n, st));
    const int* nc = c->lay.ncell;
    k_cell_flags<<<nb(n), 256, 0, st>>>(n, x, y, z, species, gas_only, c->lay.inv_q, c->lay.cs, dmask, dmask + nc[0],
                                        dmask + nc[0] + nc[1], P<uint8_t>(c->sel_flag));
    CRK_LAUNCHED(c, "cell flags");
    return compact_dev(c, n, idx_out, count_dev, st);
}

crk_status crk_select_gas_dev(crk_ctx* c, const uint8_t* dmask, int32_t* idx_out, int32_t* count_dev, void* stream) {
    if (!c || !count_dev || !dmask) return CRK_EINVAL;
    if (c->stage < ST_LISTS) return fail(c, CRK_ESTATE, "call crk_build_lists first");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t ng = c->n_gas;
    if (ng == 0) return cuda_check(c, zero_async(count_dev, 4, st, c), "memset");
    if (!idx_out) return fail(c, CRK_EINVAL, "null idx_out");
    CRK_TRY(grow(c, c->sel_flag, ng, st));
    const int* nc = c->lay.ncell;
    k_cell_flags_gas<<<nb(ng), 256, 0, st>>>(ng, P<float4>(c->gpos), c->lay.inv_q, c->lay.cs, dmask, dmask + nc[0],
                                             dmask + nc[0] + nc[1], P<uint8_t>(c->sel_flag));
    CRK_LAUNCHED(c, "gas cell flags");
    return compact_dev(c, ng, idx_out, count_dev, st);
}

crk_status crk_pack_particles_dev(crk_ctx* c, const crk_particles* p, const int32_t* idx, const int32_t* count_dev,
                                  int64_t cap, void* out, void* stream) {
    if (!c || !p || cap < 0 || !count_dev || (cap > 0 && (!idx || !out))) return fail(c, CRK_EINVAL, "bad args");
    if (cap == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    const unsigned g = nb(cap) < 4096u ? nb(cap) : 4096u;
    k_pack_particles_dev<<<g, 256, 0, (cudaStream_t)stream>>>(cap, count_dev, idx, p->x, p->y, p->z, p->vx, p->vy,
                                                              p->vz, p->m, p->H, p->u, p->species, p->id,
                                                              reinterpret_cast<Rec48*>(out));
    CRK_LAUNCHED(c, "pack particles");
    return CRK_OK;
}

crk_status crk_pack_particles(crk_ctx* c, const crk_particles* p, const int32_t* idx, int64_t n, void* out,
                              void* stream) {
    if (!c || !p || n < 0 || (n > 0 && (!idx || !out))) return fail(c, CRK_EINVAL, "bad args");
    if (n == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_pack_particles<<<nb(n), 256, 0, (cudaStream_t)stream>>>(n, idx, p->x, p->y, p->z, p->vx, p->vy, p->vz, p->m,
                                                              p->H, p->u, p->species, p->id,
                                                              reinterpret_cast<Rec48*>(out));
    CRK_LAUNCHED(c, "pack particles");
    return CRK_OK;
}

crk_status crk_unpack_particles(crk_ctx* c, crk_particles* p, int64_t offset, int64_t n, const void* in,
                                void* stream) {
    if (!c || !p || n < 0 || offset < 0 || offset + n > p->n || (n > 0 && !in)) return fail(c, CRK_EINVAL, "bad args");
    if (n == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_unpack_particles<<<nb(n), 256, 0, (cudaStream_t)stream>>>(n, offset, reinterpret_cast<const Rec48*>(in), p->x,
                                                                p->y, p->z, p->vx, p->vy, p->vz, p->m, p->H, p->u,
                                                                p->species, p->id);
    CRK_LAUNCHED(c, "unpack particles");
    return CRK_OK;
}

crk_status crk_pack_gas(crk_ctx* c, int what, const int32_t* idx, int64_t n, void* out, void* stream) {
    if (!c || (what != 0 && what != 1) || n < 0 || (n > 0 && (!idx || !out))) return fail(c, CRK_EINVAL, "bad args");
    if (what == 0 && c->stage < ST_GEO) return fail(c, CRK_ESTATE, "V is packed after crk_geometry");
    if (what == 1 && c->stage < ST_EXT) return fail(c, CRK_ESTATE, "records are packed after crk_extras");
    if (n == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_pack_gas<<<nb(what == 0 ? n : n * 9), 256, 0, (cudaStream_t)stream>>>(n, what, idx, P<float>(c->gV),
                                                                            P<float4>(c->grec), c->n_gas, out);
    CRK_LAUNCHED(c, "pack gas");
    return CRK_OK;
}

crk_status crk_pack_gas_state(crk_ctx* c, const crk_particles* p, const int32_t* idx, int64_t n, void* out,
                              void* stream) {
    if (!c || !p || !p->vx || !p->vy || !p->vz || n < 0 || (n > 0 && (!idx || !out))) return fail(c, CRK_EINVAL, "bad args");
    if (c->stage < ST_GEO) return fail(c, CRK_ESTATE, "V is packed after crk_geometry");
    if (n == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_pack_gas_state<<<nb(n), 256, 0, (cudaStream_t)stream>>>(n, idx, P<int32_t>(c->gas_idx), P<float>(c->gV), p->vx,
                                                              p->vy, p->vz, reinterpret_cast<float4*>(out));
    CRK_LAUNCHED(c, "pack gas state");
    return CRK_OK;
}

crk_status crk_unpack_gas_state(crk_ctx* c, crk_particles* p, const int32_t* idx, int64_t n, const void* in,
                                void* stream) {
    if (!c || !p || !p->vx || !p->vy || !p->vz || n < 0 || (n > 0 && (!idx || !in))) return fail(c, CRK_EINVAL, "bad args");
    if (c->stage < ST_GEO) return fail(c, CRK_ESTATE, "V is unpacked after crk_geometry");
    if (n == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_unpack_gas_state<<<nb(n), 256, 0, (cudaStream_t)stream>>>(n, idx, P<int32_t>(c->gas_idx),
                                                                reinterpret_cast<const float4*>(in), P<float4>(c->gpos),
                                                                P<float>(c->gV), P<float4>(c->gposV), p->vx, p->vy, p->vz);
    CRK_LAUNCHED(c, "unpack gas state");
    return CRK_OK;
}

crk_status crk_unpack_gas(crk_ctx* c, int what, const int32_t* idx, int64_t n, const void* in, void* stream) {
    if (!c || (what != 0 && what != 1) || n < 0 || (n > 0 && (!idx || !in))) return fail(c, CRK_EINVAL, "bad args");
    if (what == 0 && c->stage < ST_GEO) return fail(c, CRK_ESTATE, "V is unpacked after crk_geometry");
    if (what == 1 && c->stage < ST_EXT) return fail(c, CRK_ESTATE, "records are unpacked after crk_extras");
    if (n == 0) return CRK_OK;
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    k_unpack_gas<<<nb(what == 0 ? n : n * 9), 256, 0, (cudaStream_t)stream>>>(
        n, what, idx, in, P<float4>(c->gpos), P<float>(c->gV), P<float4>(c->gposV), P<float4>(c->grec), c->n_gas);
    CRK_LAUNCHED(c, "unpack gas");
    return CRK_OK;
}

}  // extern "C"
