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

// R1 selection of every peer in one pass: per particle its cell, then per peer the mask test;
// selected indices appended with one atomic per warp and peer (ballot prefix within the warp)
__global__ void k_select_peers(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                               const float* __restrict__ z, const uint8_t* __restrict__ sp, float inv_q, int cs,
                               const uint8_t* __restrict__ dmasks, int mstride, int ncx, int ncy, int npeers,
                               int32_t* __restrict__ idx_out, int64_t stride, int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31; i0 < n;
         i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + lane;
        const bool v = i < n;
        uint32_t cx = 0, cy = 0, cz = 0;
        bool gas = false;
        if (v) {
            cx = (uint32_t)(x[i] * inv_q) >> cs;
            cy = (uint32_t)(y[i] * inv_q) >> cs;
            cz = (uint32_t)(z[i] * inv_q) >> cs;
            gas = sp && sp[i] == 1;
        }
        for (int q = 0; q < npeers; ++q) {
            const uint8_t* m = dmasks + (int64_t)q * mstride;
            const bool f = v && m[cx] && m[ncx + cy] && m[ncx + ncy + cz];
            const unsigned b = __ballot_sync(0xffffffffu, f);
            if (!b) continue;
            const unsigned bg = __ballot_sync(0xffffffffu, f && gas);
            int base = 0;
            if (lane == 0) {
                base = atomicAdd(counts + 2 * q, __popc(b));
                if (bg) atomicAdd(counts + 2 * q + 1, __popc(bg));
            }
            base = __shfl_sync(0xffffffffu, base, 0);
            if (f) idx_out[q * stride + base + __popc(b & below)] = (int32_t)i;
        }
    }
}

__global__ void k_flag_own(int64_t n, const int32_t* __restrict__ perm, int64_t n_own, uint8_t* flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = perm[i] < n_own ? 1 : 0;
}

// dst row t = src row idx[t], every input field
__global__ void k_gather_rows(int64_t n, const int32_t* __restrict__ idx, const float* __restrict__ x,
                              const float* __restrict__ y, const float* __restrict__ z, const float* __restrict__ vx,
                              const float* __restrict__ vy, const float* __restrict__ vz, const float* __restrict__ m,
                              const float* __restrict__ H, const float* __restrict__ u, const uint8_t* __restrict__ sp,
                              const int64_t* __restrict__ id, float* dx, float* dy, float* dz, float* dvx, float* dvy,
                              float* dvz, float* dm, float* dH, float* du, uint8_t* dsp, int64_t* did) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t i = idx[t];
    dx[t] = x[i]; dy[t] = y[i]; dz[t] = z[i];
    dvx[t] = vx[i]; dvy[t] = vy[i]; dvz[t] = vz[i];
    dm[t] = m[i]; dH[t] = H[i]; du[t] = u[i];
    dsp[t] = sp[i];
    did[t] = id[i];
}

// ---- order-preserving selection of gas ranks for several cell-mask sets at once
// blocks of GM_B = 1024 consecutive gas ranks (8 warps x 4 sub-steps of 32); per element a bit
// per set; counts per (set, block), an exclusive scan over the blocks per set, then the writes
// at block offset + warp offset + ballot prefix, so every set's output is in ascending rank order
constexpr int GM_W = 8, GM_B = GM_W * 128, GM_MAXSETS = 16;
__device__ __forceinline__ uint32_t gm_bits(const float4* __restrict__ gpos, int64_t k, int64_t ng, float inv_q,
                                            int cs, const uint8_t* __restrict__ dm, int mstride, int ncx, int ncy,
                                            int nsets) {
    if (k >= ng) return 0u;
    const float4 p = gpos[k];
    const uint32_t cx = (uint32_t)(p.x * inv_q) >> cs, cy = (uint32_t)(p.y * inv_q) >> cs,
                   cz = (uint32_t)(p.z * inv_q) >> cs;
    uint32_t b = 0u;
    for (int q = 0; q < nsets; ++q) {
        const uint8_t* m = dm + (int64_t)q * mstride;
        if (m[cx] && m[ncx + cy] && m[ncx + ncy + cz]) b |= 1u << q;
    }
    return b;
}

__global__ void __launch_bounds__(GM_W * 32) k_gas_multi_count(int64_t ng, const float4* __restrict__ gpos, float inv_q,
                                                              int cs, const uint8_t* __restrict__ dm, int mstride,
                                                              int ncx, int ncy, int nsets, int32_t* __restrict__ blkcnt,
                                                              int64_t nblk) {
    __shared__ int s_cnt[GM_MAXSETS];
    if (threadIdx.x < GM_MAXSETS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = blockIdx.x * (int64_t)GM_B + w * 128;
    int c[GM_MAXSETS];
#pragma unroll
    for (int q = 0; q < GM_MAXSETS; ++q) c[q] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t b = gm_bits(gpos, base + 32 * j + lane, ng, inv_q, cs, dm, mstride, ncx, ncy, nsets);
#pragma unroll
        for (int q = 0; q < GM_MAXSETS; ++q)
            if (q < nsets) c[q] += __popc(__ballot_sync(0xffffffffu, (b >> q) & 1u));
    }
    if (lane == 0)
        for (int q = 0; q < nsets; ++q)
            if (c[q]) atomicAdd(&s_cnt[q], c[q]);
    __syncthreads();
    if (threadIdx.x < nsets) blkcnt[(int64_t)threadIdx.x * nblk + blockIdx.x] = s_cnt[threadIdx.x];
}

// one CTA per set: exclusive scan of its block counts (in place), the set's total to counts[q]
__global__ void __launch_bounds__(1024) k_gas_multi_scan(int32_t* __restrict__ blkcnt, int64_t nblk,
                                                        int32_t* __restrict__ counts) {
    using Scan = cub::BlockScan<int32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int32_t s_carry;
    int32_t* row = blkcnt + (int64_t)blockIdx.x * nblk;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nblk; b0 += 1024) {
        const int64_t b = b0 + threadIdx.x;
        const int32_t v = b < nblk ? row[b] : 0;
        int32_t ex, tot;
        Scan(tmp).ExclusiveSum(v, ex, tot);
        const int32_t carry = s_carry;
        if (b < nblk) row[b] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[blockIdx.x] = s_carry;
}

__global__ void __launch_bounds__(GM_W * 32) k_gas_multi_write(int64_t ng, const float4* __restrict__ gpos, float inv_q,
                                                              int cs, const uint8_t* __restrict__ dm, int mstride,
                                                              int ncx, int ncy, int nsets,
                                                              const int32_t* __restrict__ blkoff, int64_t nblk,
                                                              int32_t* __restrict__ idx_out, int64_t stride) {
    __shared__ int s_w[GM_MAXSETS][GM_W];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int64_t base = blockIdx.x * (int64_t)GM_B + w * 128;
    uint32_t bits[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bits[j] = gm_bits(gpos, base + 32 * j + lane, ng, inv_q, cs, dm, mstride, ncx, ncy, nsets);
    for (int q = 0; q < nsets; ++q) {
        int c = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) c += __popc(__ballot_sync(0xffffffffu, (bits[j] >> q) & 1u));
        if (lane == 0) s_w[q][w] = c;
    }
    __syncthreads();
    if (threadIdx.x < nsets) {  // exclusive prefix over the warps, plus the block's offset
        int run = blkoff[(int64_t)threadIdx.x * nblk + blockIdx.x];
        for (int v = 0; v < GM_W; ++v) {
            const int t = s_w[threadIdx.x][v];
            s_w[threadIdx.x][v] = run;
            run += t;
        }
    }
    __syncthreads();
    for (int q = 0; q < nsets; ++q) {
        int off = s_w[q][w];
        int32_t* out = idx_out + (int64_t)q * stride;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool f = (bits[j] >> q) & 1u;
            const unsigned b = __ballot_sync(0xffffffffu, f);
            const int pos = off + __popc(b & below);
            if (f && pos < stride) out[pos] = (int32_t)(base + 32 * j + lane);
            off += __popc(b);
        }
    }
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

crk_status crk_select_peers_dev(crk_ctx* c, const float* x, const float* y, const float* z, const uint8_t* species,
                                int64_t n, const uint8_t* dmasks, int32_t npeers, int32_t* idx_out, int64_t stride,
                                int32_t* counts_dev, void* stream) {
    if (!c || !counts_dev || !dmasks || n < 0 || npeers < 1 || npeers > 26 || stride < n ||
        (n > 0 && (!x || !y || !z || !idx_out)))
        return fail(c, CRK_EINVAL, "bad args");
    if (n >= (int64_t)1 << 31) return fail(c, CRK_ECAPACITY, "more than 2^31 particles");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    CRK_TRY(cuda_check(c, zero_async(counts_dev, (size_t)npeers * 2 * sizeof(int32_t), st, c), "memset"));
    if (n == 0) return CRK_OK;
    const int* nc = c->lay.ncell;
    int dev = c->device, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::min<int64_t>(nb(n), (int64_t)nsm * 8);
    k_select_peers<<<(unsigned)blocks, 256, 0, st>>>(n, x, y, z, species, c->lay.inv_q, c->lay.cs, dmasks,
                                                     nc[0] + nc[1] + nc[2], nc[0], nc[1], npeers, idx_out, stride,
                                                     counts_dev);
    CRK_LAUNCHED(c, "select peers");
    return CRK_OK;
}

crk_status crk_compact_own(crk_ctx* c, const crk_particles* src, int64_t n_own, crk_particles* dst, void* stream) {
    if (!c || !src || !dst || n_own < 0 || n_own > src->n) return fail(c, CRK_EINVAL, "bad args");
    if (n_own == 0) return CRK_OK;
    const crk_particles* both[2] = {src, dst};
    for (const crk_particles* q : both) {
        const void* f[] = {q->x, q->y, q->z, q->vx, q->vy, q->vz, q->m, q->H, q->u, q->species, q->id};
        for (const void* ptr : f)
            if (!ptr) return fail(c, CRK_EINVAL, "null input field");
    }
    if (!src->perm) return fail(c, CRK_EINVAL, "null perm (call crk_build_lists on src first)");
    if (src->n >= (int64_t)1 << 31) return fail(c, CRK_ECAPACITY, "more than 2^31 particles");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = src->n;
    CRK_TRY(grow(c, c->sel_flag, n, st));
    CRK_TRY(grow(c, c->idx_a, n * 4, st));  // build scratch, free between builds
    k_flag_own<<<nb(n), 256, 0, st>>>(n, src->perm, n_own, P<uint8_t>(c->sel_flag));
    CRK_LAUNCHED(c, "flag own");
    CRK_TRY(grow(c, c->dev_scalars, 64, st));
    CRK_TRY(compact_dev(c, n, P<int32_t>(c->idx_a), reinterpret_cast<int32_t*>(P<char>(c->dev_scalars) + 48), st));
    k_gather_rows<<<nb(n_own), 256, 0, st>>>(n_own, P<int32_t>(c->idx_a), src->x, src->y, src->z, src->vx, src->vy,
                                             src->vz, src->m, src->H, src->u, src->species, src->id, dst->x, dst->y,
                                             dst->z, dst->vx, dst->vy, dst->vz, dst->m, dst->H, dst->u, dst->species,
                                             dst->id);
    CRK_LAUNCHED(c, "gather own");
    return CRK_OK;
}

crk_status crk_select_gas_multi_dev(crk_ctx* c, const uint8_t* dmasks, int32_t nsets, int32_t* idx_out, int64_t stride,
                                    int32_t* counts_dev, void* stream) {
    if (!c || !dmasks || !counts_dev || nsets < 1 || nsets > GM_MAXSETS) return fail(c, CRK_EINVAL, "bad args");
    if (c->stage < ST_LISTS) return fail(c, CRK_ESTATE, "call crk_build_lists first");
    const int64_t ng = c->n_gas;
    if (stride < 0 || (ng > 0 && stride > 0 && !idx_out)) return fail(c, CRK_EINVAL, "bad idx_out / stride");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    cudaStream_t st = (cudaStream_t)stream;
    if (ng == 0) return cuda_check(c, zero_async(counts_dev, (size_t)nsets * 4, st, c), "memset");
    const int64_t nblk = (ng + GM_B - 1) / GM_B;
    CRK_TRY(grow(c, c->sel_flag, (size_t)nsets * nblk * 4, st));  // block counts -> offsets
    int32_t* blk = P<int32_t>(c->sel_flag);
    const int* nc = c->lay.ncell;
    const int ms = nc[0] + nc[1] + nc[2];
    k_gas_multi_count<<<(unsigned)nblk, GM_W * 32, 0, st>>>(ng, P<float4>(c->gpos), c->lay.inv_q, c->lay.cs, dmasks, ms,
                                                            nc[0], nc[1], nsets, blk, nblk);
    CRK_LAUNCHED(c, "gas multi count");
    k_gas_multi_scan<<<(unsigned)nsets, 1024, 0, st>>>(blk, nblk, counts_dev);
    CRK_LAUNCHED(c, "gas multi scan");
    k_gas_multi_write<<<(unsigned)nblk, GM_W * 32, 0, st>>>(ng, P<float4>(c->gpos), c->lay.inv_q, c->lay.cs, dmasks, ms,
                                                            nc[0], nc[1], nsets, blk, nblk, idx_out, stride);
    CRK_LAUNCHED(c, "gas multi write");
    return CRK_OK;
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
