// build.cu — a1 + a2: sort, leaf build and leaf-pair interaction lists
// (definitions §8(c) O1, O3, O4; the paper's leaves: PAPER.md:418-422).
//
//   key (cell Morton | in-cell Morton) -> CUB onesweep radix sort (+ id tie fix)
//   -> permute the caller's SoA in place -> chaining-mesh cell runs (dense, Morton-indexed)
//   -> gas ranks -> four leaf sets (balanced chunks of each cell run) -> bboxes
//   -> gravity and hydro CSR lists (exact fp64 bbox test, per-axis periodic shift).
// HBM-bound; every kernel is a streaming pass except the list kernels (one warp per i-leaf).
#include <cub/cub.cuh>

#include <cstring>
#include <cmath>
#include "common.cuh"

namespace crk {

// ---------------------------------------------------------------- keys
// 32-bit key = Morton(cell) << 3 fbits | Morton(top fbits of the in-cell coordinate) (O3)
// Also packs each particle (input order) into a 48-byte record, so that the permutation
// gathers one record per particle (two sectors) instead of eleven scattered fields — the
// difference between 0.5 and 7.6 ms on a randomly ordered input (c4).
struct SoA {
    float* f[9];       // x y z vx vy vz m H u
    uint8_t* sp;
    int64_t* id;
};

__global__ void k_keys(int64_t n, SoA in, float inv_q, int cs, int fbits, uint32_t* keys, int32_t* idx,
                       float4* rec, int32_t* ccount) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x = in.f[0][i], y = in.f[1][i], z = in.f[2][i];
    const int64_t id = in.id[i];
    rec[3 * i] = make_float4(x, y, z, in.f[3][i]);
    rec[3 * i + 1] = make_float4(in.f[4][i], in.f[5][i], in.f[6][i], in.f[7][i]);
    rec[3 * i + 2] = make_float4(in.f[8][i], __int_as_float((int)in.sp[i]), __int_as_float((int)(uint32_t)id),
                                 __int_as_float((int)(uint32_t)((uint64_t)id >> 32)));
    const uint32_t xi = (uint32_t)(x * inv_q), yi = (uint32_t)(y * inv_q), zi = (uint32_t)(z * inv_q);
    const uint32_t msk = (1u << cs) - 1u, sh = cs - fbits;
    const uint64_t cm = morton3(xi >> cs, yi >> cs, zi >> cs);
    const uint64_t fm = morton3((xi & msk) >> sh, (yi & msk) >> sh, (zi & msk) >> sh);
    keys[i] = (uint32_t)((cm << (3 * fbits)) | fm);
    idx[i] = (int32_t)i;
    // cell histogram, one atomic per run of equal cells in the warp (sorted inputs: ~1 per warp)
    const unsigned same = __match_any_sync(__activemask(), (uint32_t)cm);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(ccount + cm, __popc(same));
}

// counting sort by cell: each particle's slot in its cell's range (order within a cell arbitrary;
// the per-cell sort by the in-cell key and the id tie fix make the order total, O3)
__global__ void k_cell_scatter(int64_t n, const uint32_t* __restrict__ keys, int fbits, const int32_t* __restrict__ coff,
                               int32_t* cursor, uint32_t* keys_out, int32_t* idx_out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t key = keys[i];
    const uint32_t cell = key >> (3 * fbits);
    const unsigned same = __match_any_sync(__activemask(), cell);
    const int lane = threadIdx.x & 31, leader = __ffs(same) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(cursor + cell, __popc(same));
    base = __shfl_sync(same, base, leader);
    const int pos = coff[cell] + base + __popc(same & ((1u << lane) - 1u));
    keys_out[pos] = key;
    idx_out[pos] = (int32_t)i;
}

// lanes holding the same 6-bit digit (65 for none): the classic multisplit from 7 ballots
__device__ __forceinline__ unsigned same_digit_lanes(uint32_t d) {
    unsigned m = __ballot_sync(0xffffffffu, d < 64u);
    m = d < 64u ? m : ~m;
#pragma unroll
    for (int b = 0; b < 6; ++b) {
        const unsigned q = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? q : ~q;
    }
    return m;
}
// per-cell sort of the cell-scattered keys by their in-cell bits (3 fbits): one warp per cell, an LSD
// radix sort in shared memory, 6 bits per pass, each pass stable (ranks from ballots in input
// order); equal keys keep the scatter's order and k_tie_fix then orders them by id (O3).
// Cells of more than CELL_SORT_MAX particles get a segment in (beg, end) for CUB's segmented sort
// (clustered inputs), the others an empty one.
constexpr int CELL_SORT_MAX = 256;
__global__ void __launch_bounds__(256) k_cell_sort(int64_t ncm, int fine_bits, const int32_t* __restrict__ coff,
                                                   const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ idx_in,
                                                   uint32_t* keys_out, int32_t* idx_out, int32_t* beg, int32_t* end,
                                                   int* nbig) {
    __shared__ uint2 s[8][2][CELL_SORT_MAX];  // (key, index), double buffer
    __shared__ int cnt[8][64];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int64_t c = blockIdx.x * 8 + w;
    if (c >= ncm) return;
    const int o = coff[c], nc = coff[c + 1] - o;
    const bool big = nc > CELL_SORT_MAX;
    if (lane == 0) {
        beg[c] = big ? o : 0;
        end[c] = big ? o + nc : 0;
        if (big) atomicAdd(nbig, 1);
    }
    if (big || nc == 0) return;
    uint2* src = s[w][0];
    uint2* dst = s[w][1];
    for (int t = lane; t < nc; t += 32) src[t] = make_uint2(keys_in[o + t], (uint32_t)idx_in[o + t]);
    __syncwarp();
    for (int sh = 0; sh < fine_bits; sh += 6) {
        cnt[w][lane] = 0;
        cnt[w][lane + 32] = 0;
        __syncwarp();
        for (int t0 = 0; t0 < nc; t0 += 32) {  // histogram
            const int t = t0 + lane;
            const uint32_t d = t < nc ? (src[t].x >> sh) & 63u : 64u;
            if (d < 64u) atomicAdd(&cnt[w][d], 1);
        }
        __syncwarp();
        // exclusive scan of the 64 counts (two per lane)
        const int c0 = cnt[w][2 * lane], c1 = cnt[w][2 * lane + 1];
        int x = c0 + c1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        __syncwarp();
        cnt[w][2 * lane] = x - c0 - c1;
        cnt[w][2 * lane + 1] = x - c1;
        __syncwarp();
        for (int t0 = 0; t0 < nc; t0 += 32) {  // stable scatter
            const int t = t0 + lane;
            const uint2 v = t < nc ? src[t] : make_uint2(0u, 0u);
            const uint32_t d = t < nc ? (v.x >> sh) & 63u : 64u;
            const unsigned same = same_digit_lanes(d);
            const int base = d < 64u ? cnt[w][d] : 0;
            if (d < 64u) dst[base + __popc(same & below)] = v;
            __syncwarp();
            if (d < 64u && lane == __ffs(same) - 1) cnt[w][d] = base + __popc(same);
            __syncwarp();
        }
        uint2* tsw = src; src = dst; dst = tsw;
    }
    for (int t = lane; t < nc; t += 32) {
        const uint2 v = src[t];
        keys_out[o + t] = v.x;
        idx_out[o + t] = (int32_t)v.y;
    }
}

// Runs of equal keys (coincident to 1/2^fbits of a cell) are ordered by id: total order (O3).
__global__ void k_tie_fix(int64_t n, const uint32_t* __restrict__ keys, int32_t* idx, const int64_t* __restrict__ id) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k + 1 >= n) return;
    if (keys[k] != keys[k + 1]) return;
    if (k > 0 && keys[k - 1] == keys[k]) return;  // not the run start
    int64_t e = k + 1;
    while (e + 1 < n && keys[e + 1] == keys[k]) ++e;
    for (int64_t a = k + 1; a <= e; ++a) {  // insertion sort by id
        const int32_t v = idx[a];
        const int64_t iv = id[v];
        int64_t b = a - 1;
        while (b >= k && id[idx[b]] > iv) {
            idx[b + 1] = idx[b];
            --b;
        }
        idx[b + 1] = v;
    }
}

// ---------------------------------------------------------------- permute (one gather pass)

// gather the packed records in sorted order straight into the caller's arrays (the records
// are a copy, so this is safe in place) and derive xm, gas flags and cell runs
__global__ void k_permute(int64_t n, const int32_t* __restrict__ perm, const float4* __restrict__ rec, SoA dst,
                          const uint32_t* __restrict__ keys, int fbits, float4* xm, int32_t* gflag, int32_t* cstart,
                          int32_t* cend, int32_t* perm_out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t s = perm[k];
    if (perm_out) perm_out[k] = (int32_t)s;
    const float4 r0 = __ldg(rec + 3 * s), r1 = __ldg(rec + 3 * s + 1), r2 = __ldg(rec + 3 * s + 2);
    dst.f[0][k] = r0.x; dst.f[1][k] = r0.y; dst.f[2][k] = r0.z; dst.f[3][k] = r0.w;
    dst.f[4][k] = r1.x; dst.f[5][k] = r1.y; dst.f[6][k] = r1.z; dst.f[7][k] = r1.w;
    dst.f[8][k] = r2.x;
    const int sp = __float_as_int(r2.y);
    dst.sp[k] = (uint8_t)sp;
    dst.id[k] = (int64_t)(((uint64_t)(uint32_t)__float_as_int(r2.w) << 32) | (uint32_t)__float_as_int(r2.z));
    xm[k] = make_float4(r0.x, r0.y, r0.z, r1.z);
    gflag[k] = sp == 1 ? 1 : 0;
    const uint32_t c = keys[k] >> (3 * fbits);
    if (k == 0 || (keys[k - 1] >> (3 * fbits)) != c) cstart[c] = (int32_t)k;
    if (k == n - 1 || (keys[k + 1] >> (3 * fbits)) != c) cend[c] = (int32_t)(k + 1);
}

__global__ void k_gas_pack(int64_t n, const int32_t* __restrict__ gflag, const int32_t* __restrict__ grank,
                           const float4* __restrict__ xm, const float* __restrict__ H, int32_t* gas_idx, float4* gpos,
                           float* dmax_h2) {
    __shared__ float wmax[32];
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float h2 = 0.f;
    if (k < n && gflag[k]) {
        const int32_t g = grank[k];
        gas_idx[g] = (int32_t)k;
        const float4 p = xm[k];
        const float h = H[k];
        gpos[g] = make_float4(p.x, p.y, p.z, h);
        h2 = __fmul_rn(h, h);
    }
    h2 = warp_max(h2);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = h2;
    __syncthreads();
    if (threadIdx.x < 32) {
        h2 = threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0.f;
        h2 = warp_max(h2);
        if (threadIdx.x == 0 && h2 > 0.f) atomicMax(reinterpret_cast<int*>(dmax_h2), __float_as_int(h2));
    }
}

// ---------------------------------------------------------------- leaves (O3)
// counts per cell for the 4 leaf sets: cnt[s*(ncm+1) + c]
struct Dom {
    int lo[3], hi[3];
};
// is Morton-indexed cell c owned by this domain?
__device__ __forceinline__ bool owned(uint64_t c, const Dom& d) {
    const int cx = (int)compact3(c), cy = (int)compact3(c >> 1), cz = (int)compact3(c >> 2);
    return cx >= d.lo[0] && cx < d.hi[0] && cy >= d.lo[1] && cy < d.hi[1] && cz >= d.lo[2] && cz < d.hi[2];
}

// i-leaf sets (0, 2) only in owned cells; j-leaf sets (1, 3) in every populated cell
__global__ void k_leaf_counts(int64_t ncm, const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                              const int32_t* __restrict__ grank, int l0, int l1, int l2, int l3, Dom dom,
                              int32_t* cnt) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c > ncm) return;
    int nc = 0, gc = 0;
    bool own = false;
    if (c < ncm) {
        nc = cend[c] - cstart[c];
        if (nc > 0) gc = grank[cend[c]] - grank[cstart[c]];
        own = owned((uint64_t)c, dom);
    }
    cnt[0 * (ncm + 1) + c] = own ? (nc + l0 - 1) / l0 : 0;
    cnt[1 * (ncm + 1) + c] = (nc + l1 - 1) / l1;
    cnt[2 * (ncm + 1) + c] = own ? (gc + l2 - 1) / l2 : 0;
    cnt[3 * (ncm + 1) + c] = (gc + l3 - 1) / l3;
}

__global__ void k_leaf_fill(int64_t ncm, const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                            const int32_t* __restrict__ grank, const int32_t* __restrict__ off, int set, int lmax,
                            Dom dom, int32_t* first, int32_t* count, uint64_t* lcell) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncm) return;
    const int nc = cend[c] - cstart[c];
    if (nc <= 0) return;
    if ((set == 0 || set == 2) && !owned((uint64_t)c, dom)) return;
    int base, cnt;
    if (set < 2) {
        base = cstart[c];
        cnt = nc;
    } else {
        base = grank[cstart[c]];
        cnt = grank[cend[c]] - base;
    }
    const int nch = (cnt + lmax - 1) / lmax;
    const int o = off[c];
    for (int t = 0; t < nch; ++t) {
        const int lo = (int)((int64_t)t * cnt / nch), hi = (int)((int64_t)(t + 1) * cnt / nch);
        first[o + t] = base + lo;
        count[o + t] = hi - lo;
        lcell[o + t] = (uint64_t)c;
    }
}

// bbox (+ max H^2) of big leaves (i-leaf sets): one warp per leaf, lanes stride the members
__global__ void k_leaf_bbox_warp(int64_t nl, const int32_t* __restrict__ first, const int32_t* __restrict__ count,
                                 const float4* __restrict__ pts, int gas, float* bbox, float* maxh2, float4* box8) {
    const int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (l >= nl) return;
    float lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY, mh = 0.f;
    const int f = first[l], c = count[l];
    for (int t = lane; t < c; t += 32) {
        const float4 p = pts[f + t];
        lo0 = fminf(lo0, p.x); lo1 = fminf(lo1, p.y); lo2 = fminf(lo2, p.z);
        hi0 = fmaxf(hi0, p.x); hi1 = fmaxf(hi1, p.y); hi2 = fmaxf(hi2, p.z);
        if (gas) mh = fmaxf(mh, __fmul_rn(p.w, p.w));
    }
    lo0 = warp_min(lo0); lo1 = warp_min(lo1); lo2 = warp_min(lo2);
    hi0 = warp_max(hi0); hi1 = warp_max(hi1); hi2 = warp_max(hi2);
    mh = warp_max(mh);
    if (lane == 0) {
        float* b = bbox + 6 * l;
        b[0] = lo0; b[1] = lo1; b[2] = lo2; b[3] = hi0; b[4] = hi1; b[5] = hi2;
        if (gas) maxh2[l] = mh;
        box8[2 * l] = make_float4(lo0, lo1, lo2, mh);
        box8[2 * l + 1] = make_float4(hi0, hi1, hi2, 0.f);
    }
}

// bbox (+ max H^2) per leaf; one thread per leaf, members contiguous in xm / gpos
__global__ void k_leaf_bbox(int64_t nl, const int32_t* __restrict__ first, const int32_t* __restrict__ count,
                            const float4* __restrict__ pts, int gas, float* bbox, float* maxh2, float4* box8) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= nl) return;
    float lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY, mh = 0.f;
    const int f = first[l], c = count[l];
    for (int t = 0; t < c; ++t) {
        const float4 p = pts[f + t];
        lo0 = fminf(lo0, p.x); lo1 = fminf(lo1, p.y); lo2 = fminf(lo2, p.z);
        hi0 = fmaxf(hi0, p.x); hi1 = fmaxf(hi1, p.y); hi2 = fmaxf(hi2, p.z);
        if (gas) mh = fmaxf(mh, __fmul_rn(p.w, p.w));
    }
    float* b = bbox + 6 * l;
    b[0] = lo0; b[1] = lo1; b[2] = lo2; b[3] = hi0; b[4] = hi1; b[5] = hi2;
    if (gas) maxh2[l] = mh;
    box8[2 * l] = make_float4(lo0, lo1, lo2, mh);  // 32-byte padded copy for TMA staging
    box8[2 * l + 1] = make_float4(hi0, hi1, hi2, 0.f);
}

// ---------------------------------------------------------------- lists (O4)
// per axis: gap_s = max(0, lo_b + sL - hi_a, lo_a - hi_b - sL) for s = 0, -1, +1 (first
// minimum); d2 = sum gap^2 in fp64 (exact for q-multiples); keep iff d2 < cut2 (1 + 2^-20).
__device__ __forceinline__ bool leaf_pair_test(const float* ba, const float* bb, const double L[3], double cut2s,
                                               int& code) {
    double d2 = 0.0;
    int sc[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double best = 1e300;
        int bs = 0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int s = t == 0 ? 0 : (t == 1 ? -1 : 1);
            const double sL = s * L[d];
            const double g1 = (double)bb[d] + sL - (double)ba[3 + d];
            const double g2 = (double)ba[d] - (double)bb[3 + d] - sL;
            const double g = fmax(0.0, fmax(g1, g2));
            if (g < best) { best = g; bs = s; }
        }
        sc[d] = bs;
        d2 = fma(best, best, d2);  // exact: all terms are integers times q^2 below 2^52 q^2
    }
    code = (sc[0] + 1) + 3 * (sc[1] + 1) + 9 * (sc[2] + 1);
    return d2 < cut2s;
}

struct ListArgs {
    int64_t nA;
    const float* bboxA;
    const float* maxh2A;
    const float* bboxB;
    const float* maxh2B;
    const int32_t* loffB;  // per-cell offsets of the j-leaf set (ncm + 1)
    const float* dmax_h2;  // global max H^2 (hydro mode)
    int mode;              // 0 gravity (rcut2), 1 hydro (max of the two leaves' max H^2)
    float rcut2;
    double L[3];
    float Lf[3];
    double cell_side;
    float inv_q;
    double q2inv_slack;    // (1 + 2^-20) / q^2, exact
    int ncell[3];
    int32_t* rowlen;       // bound pass: candidate j-leaves per row (upper bound of its length)
    const int32_t* rowoff; // fill pass: where each row starts (exclusive scan of the bounds)
    int32_t* rowend;       // fill pass: where each row ends
    const int32_t* jfirst;  // j-leaf first member / count (packed entry records)
    const int32_t* jcount;
    int2* erec;
    const float4* box8B;    // padded j-leaf boxes (lo, max H^2), (hi, 0)
    double skin;            // list skin: cutoffs sqrt(cut2) + skin (0: the exact O4 lists)
    uint8_t* rclass;        // fill pass, hydro lists of a partial domain (else null): 1 = the row holds a ghost j-leaf
    int dlo[3], dhi[3];     // owned cells [dlo, dhi)
};

// ---------------------------------------------------------------- gravity entry masks
// Bit g of a gravity entry's mask is set iff the entry's j-leaf can hold a pair for i-group g of
// the row's leaf (i-particles [first + 16g, first + 16g + 16)): the leaf reaches past the
// group's first particle (Newton-3: pairs with j below the group belong to an earlier group) or
// is a ghost (no group of its own on this rank), and the fp32 box-box distance of the group's
// bounding box to the shifted j-leaf box is below rcut2 * CULL_SLACK (a superset of O2).  This
// is grav_pipe_kernel's entry cull, computed once per entry by the list build (and again by
// crk_refresh) instead of by every group's warp over the whole row.
// group bounding boxes of leaf (f0, cnt <= 128) into gb[8][6] (lo xyz, hi xyz); one warp
__device__ __forceinline__ void group_boxes(const float4* __restrict__ xm, int f0, int cnt, float (*gb)[6], int lane) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int k = lane + 32 * t;  // group 2t + lane / 16
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        if (k < cnt) {
            const float4 p = xm[f0 + k];
            lo[0] = hi[0] = p.x; lo[1] = hi[1] = p.y; lo[2] = hi[2] = p.z;
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
                hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
            }
        if ((lane & 15) == 0)
#pragma unroll
            for (int d = 0; d < 3; ++d) { gb[2 * t + lane / 16][d] = lo[d]; gb[2 * t + lane / 16][3 + d] = hi[d]; }
    }
    __syncwarp();
}
// a j-leaf lies in one cell: its (unshifted) box centre decides whether it is a ghost
__device__ __forceinline__ bool leaf_ghost(const float4& bl, const float4& bh, float inv_q, int cs, const int* dlo,
                                           const int* dhi) {
    const int cx = (int)(0.5f * (bl.x + bh.x) * inv_q) >> cs, cy = (int)(0.5f * (bl.y + bh.y) * inv_q) >> cs,
              cz = (int)(0.5f * (bl.z + bh.z) * inv_q) >> cs;
    return !(cx >= dlo[0] && cx < dhi[0] && cy >= dlo[1] && cy < dhi[1] && cz >= dlo[2] && cz < dhi[2]);
}

// cut^2 of the O4 test with the skin: (sqrt(cut2) + skin)^2 (the plain cut2 without one)
__device__ __forceinline__ double skin_cut2(double cut2, double skin) {
    if (skin <= 0.0) return cut2;
    const double c = sqrt(cut2) + skin;
    return c * c;
}

__device__ __forceinline__ void put_entry(const ListArgs& A, int p, int b, int code) {
    // (the CSR col / shift views of crk_list_view are decoded from erec on demand)
    A.erec[p] = make_int2(A.jfirst[b] | ((A.jcount[b] - 1) << 29), b | (code << 26));
}

constexpr int LIST_WARPS = 8;

// One warp per i-leaf.  Fast path (the usual case): the candidate cells around the
// i-bbox do not wrap onto themselves, so each cell's periodic shift is known from the
// wrap; cells whose box is out of reach are pruned; the j-leaves of the surviving
// cells are flattened across the lanes (warp scan) and tested with the exact integer
// form of O4 (gaps are multiples of q below 2^24 q).  Tiny boxes use the generic path
// with the per-axis shift search.
// Two launches: FILL = false only sums the candidate j-leaves of the surviving cells (an
// upper bound of the row's length: no leaf tests), FILL = true tests and writes the row at the
// start its bound reserved and records where it ends — one pass of leaf tests instead of a
// count pass and a fill pass.
template <bool FILL>
__global__ void __launch_bounds__(LIST_WARPS * 32, 5) k_lists(ListArgs A) {
    __shared__ int32_t s_b0[LIST_WARPS][32], s_ex[LIST_WARPS][32], s_code[LIST_WARPS][32];
    const int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    if (a >= A.nA) return;

    const float* ba = A.bboxA + 6 * a;
    const double slack = 1.0 + 0x1p-20;
    double reach2;
    if (A.mode == 0) reach2 = (double)A.rcut2;
    else reach2 = fmax((double)A.maxh2A[a], (double)*A.dmax_h2);
    reach2 = skin_cut2(reach2, A.skin);
    const double reach = sqrt(reach2 * slack) * (1.0 + 1e-12) + 1e-12;
    int c0[3], c1[3];
    bool generic = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        c0[d] = (int)floor(((double)ba[d] - reach) / A.cell_side);
        c1[d] = (int)floor(((double)ba[3 + d] + reach) / A.cell_side);
        if (c1[d] - c0[d] + 1 >= A.ncell[d]) { c0[d] = 0; c1[d] = A.ncell[d] - 1; generic = true; }
    }
    int outpos = FILL ? A.rowoff[a] : 0;
    int total = 0;
    bool ghost_ref = false;  // (hydro fill of a partial domain) some candidate j-leaf is a ghost
    const float mh2a = A.mode == 1 ? A.maxh2A[a] : 0.f;
    if (!generic) {
        const int nx = c1[0] - c0[0] + 1, ny = c1[1] - c0[1] + 1, nz = c1[2] - c0[2] + 1;
        const int ncand = nx * ny * nz;
        const double cs = A.cell_side;
        for (int cb = 0; cb < ncand; cb += 32) {
            const int t = cb + lane;
            int nb = 0, b0 = 0, code = 13;
            if (t < ncand) {
                const int ix = t % nx, iy = (t / nx) % ny, iz = t / (nx * ny);
                const int cc[3] = {c0[0] + ix, c0[1] + iy, c0[2] + iz};
                double d2c = 0.0;
                int wc[3], sc[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double lo = cc[d] * cs, hi = lo + cs;
                    const double g = fmax(0.0, fmax(lo - (double)ba[3 + d], (double)ba[d] - hi));
                    d2c += g * g;
                    wc[d] = cc[d] < 0 ? cc[d] + A.ncell[d] : (cc[d] >= A.ncell[d] ? cc[d] - A.ncell[d] : cc[d]);
                    sc[d] = cc[d] < 0 ? -1 : (cc[d] >= A.ncell[d] ? 1 : 0);
                }
                if (d2c < reach2 * slack) {
                    const uint64_t m = morton3((uint32_t)wc[0], (uint32_t)wc[1], (uint32_t)wc[2]);
                    b0 = A.loffB[m];
                    nb = A.loffB[m + 1] - b0;
                    code = (sc[0] + 1) + 3 * (sc[1] + 1) + 9 * (sc[2] + 1);
                    if (FILL && A.rclass && nb > 0)  // a ghost cell (conservative: before the leaf tests)
                        ghost_ref |= !(wc[0] >= A.dlo[0] && wc[0] < A.dhi[0] && wc[1] >= A.dlo[1] && wc[1] < A.dhi[1] &&
                                       wc[2] >= A.dlo[2] && wc[2] < A.dhi[2]);
                }
            }
            int pre = nb;  // inclusive warp scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= o) pre += v;
            }
            const int tot = __shfl_sync(0xffffffffu, pre, 31);
            if (!FILL) {  // bound: every candidate leaf of the surviving cells
                total += tot;
                continue;
            }
            s_b0[w][lane] = b0;
            s_ex[w][lane] = pre - nb;
            s_code[w][lane] = code;
            __syncwarp();
            for (int u0 = 0; u0 < tot; u0 += 32) {
                const int u = u0 + lane;
                bool keep = false;
                int b = 0, cd = 13;
                if (u < tot) {
                    int lo = 0, hi = 31;
#pragma unroll
                    for (int it = 0; it < 5; ++it) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_ex[w][mid] <= u) lo = mid; else hi = mid - 1;
                    }
                    b = s_b0[w][lo] + (u - s_ex[w][lo]);
                    cd = s_code[w][lo];
                    const float4 blo = __ldg(A.box8B + 2 * (int64_t)b), bhi = __ldg(A.box8B + 2 * (int64_t)b + 1);
                    const float bb[6] = {blo.x, blo.y, blo.z, bhi.x, bhi.y, bhi.z};
                    int sx, sy, sz;
                    decode_shift(cd, sx, sy, sz);
                    const float sL[3] = {(float)sx * A.Lf[0], (float)sy * A.Lf[1], (float)sz * A.Lf[2]};
                    uint64_t K = 0;
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const float g1 = (bb[d] + sL[d]) - ba[3 + d];   // exact (O1)
                        const float g2 = ba[d] - (bb[3 + d] + sL[d]);
                        const float g = fmaxf(0.f, fmaxf(g1, g2));
                        const uint32_t k = (uint32_t)(g * A.inv_q);     // exact integer < 2^24
                        K += (uint64_t)k * k;
                    }
                    const float cut2 = A.mode == 0 ? A.rcut2 : fmaxf(mh2a, blo.w);
                    keep = (double)K < skin_cut2((double)cut2, A.skin) * A.q2inv_slack;
                }
                const unsigned msk = __ballot_sync(0xffffffffu, keep);
                if (FILL && keep) put_entry(A, outpos + __popc(msk & ((1u << lane) - 1u)), b, cd);
                outpos += __popc(msk);
                total += __popc(msk);
            }
            __syncwarp();
        }
    } else {
        for (int cz = c0[2]; cz <= c1[2]; ++cz)
            for (int cy = c0[1]; cy <= c1[1]; ++cy)
                for (int cx = c0[0]; cx <= c1[0]; ++cx) {
                    const uint32_t wx = (uint32_t)((cx % A.ncell[0] + A.ncell[0]) % A.ncell[0]);
                    const uint32_t wy = (uint32_t)((cy % A.ncell[1] + A.ncell[1]) % A.ncell[1]);
                    const uint32_t wz = (uint32_t)((cz % A.ncell[2] + A.ncell[2]) % A.ncell[2]);
                    const uint64_t m = morton3(wx, wy, wz);
                    const int b0 = A.loffB[m], b1 = A.loffB[m + 1];
                    if (FILL && A.rclass && b1 > b0)
                        ghost_ref |= !((int)wx >= A.dlo[0] && (int)wx < A.dhi[0] && (int)wy >= A.dlo[1] &&
                                       (int)wy < A.dhi[1] && (int)wz >= A.dlo[2] && (int)wz < A.dhi[2]);
                    if (!FILL) {
                        total += b1 - b0;
                        continue;
                    }
                    for (int bb = b0; bb < b1; bb += 32) {
                        const int b = bb + lane;
                        bool keep = false;
                        int code = 13;
                        if (b < b1) {
                            const double cut2 = A.mode == 0 ? (double)A.rcut2
                                                            : fmax((double)mh2a, (double)A.maxh2B[b]);
                            keep = leaf_pair_test(ba, A.bboxB + 6 * (int64_t)b, A.L, skin_cut2(cut2, A.skin) * slack,
                                                  code);
                        }
                        const unsigned msk = __ballot_sync(0xffffffffu, keep);
                        if (FILL && keep) put_entry(A, outpos + __popc(msk & ((1u << lane) - 1u)), b, code);
                        outpos += __popc(msk);
                        total += __popc(msk);
                    }
                }
    }
    if (FILL && A.rclass) ghost_ref = __any_sync(0xffffffffu, ghost_ref);
    if (lane == 0) {
        if (FILL) A.rowend[a] = outpos;
        else A.rowlen[a] = total;
        if (FILL && A.rclass) A.rclass[a] = ghost_ref ? 1 : 0;
    }
}

// ---------------------------------------------------------------- driver
static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

static bool want_masks(const crk_ctx* c) {  // only the pipelined Newton-3 kernel (grav_kernel 0-2) reads them
    return (c->prm.symmetric & 1) && c->prm.grav_kernel <= 2;
}

static ListArgs list_args(crk_ctx* c, int m) {
    const Layout& L = c->lay;
    const int sa = m == 0 ? 0 : 2, sb = m == 0 ? 1 : 3;
    ListArgs A;
    A.nA = c->nleaf[sa];
    A.bboxA = P<float>(c->lbbox[sa]);
    A.maxh2A = sa >= 2 ? P<float>(c->lmaxh2[sa]) : nullptr;
    A.bboxB = P<float>(c->lbbox[sb]);
    A.maxh2B = sb >= 2 ? P<float>(c->lmaxh2[sb]) : nullptr;
    A.loffB = P<int32_t>(c->leaf_cnt) + sb * (L.ncm + 1);
    A.dmax_h2 = P<float>(c->dev_scalars);
    A.mode = m;
    A.rcut2 = c->prm.rcut2;
    for (int d = 0; d < 3; ++d) {
        A.L[d] = c->prm.box[d];
        A.Lf[d] = (float)c->prm.box[d];
        A.ncell[d] = L.ncell[d];
    }
    A.cell_side = c->prm.cell_side;
    A.inv_q = L.inv_q;
    A.q2inv_slack = (1.0 + 0x1p-20) / (L.q * L.q);
    A.rowlen = P<int32_t>(c->rowlen[m]);
    A.rowoff = P<int32_t>(c->rowoff[m]);
    A.rowend = P<int32_t>(c->rowend[m]);
    A.jfirst = P<int32_t>(c->lfirst[sb]);
    A.rclass = (m == 1 && L.partial) ? P<uint8_t>(c->rclass) : nullptr;
    for (int d = 0; d < 3; ++d) { A.dlo[d] = L.dlo[d]; A.dhi[d] = L.dhi[d]; }
    A.jcount = P<int32_t>(c->lcount[sb]);
    A.erec = P<int2>(c->erec[m]);
    A.box8B = P<float4>(c->lbox8[sb]);
    A.skin = c->prm.skin;
    return A;
}

// per-leaf boxes of leaf set s from the packed positions (xm: gravity sets, gpos: gas sets)
static crk_status leaf_boxes(crk_ctx* c, int s, cudaStream_t st) {
    if (c->nleaf[s] > 0 && (s == 0 || s == 2)) {
        k_leaf_bbox_warp<<<nblk(c->nleaf[s] * 32, 256), 256, 0, st>>>(
            c->nleaf[s], P<int32_t>(c->lfirst[s]), P<int32_t>(c->lcount[s]),
            s < 2 ? P<float4>(c->xm) : P<float4>(c->gpos), s >= 2, P<float>(c->lbbox[s]),
            s >= 2 ? P<float>(c->lmaxh2[s]) : nullptr, P<float4>(c->lbox8[s]));
        CRK_LAUNCHED(c, "leaf bbox");
    } else if (c->nleaf[s] > 0) {
        k_leaf_bbox<<<nblk(c->nleaf[s], 128), 128, 0, st>>>(
            c->nleaf[s], P<int32_t>(c->lfirst[s]), P<int32_t>(c->lcount[s]),
            s < 2 ? P<float4>(c->xm) : P<float4>(c->gpos), s >= 2, P<float>(c->lbbox[s]),
            s >= 2 ? P<float>(c->lmaxh2[s]) : nullptr, P<float4>(c->lbox8[s]));
        CRK_LAUNCHED(c, "leaf bbox");
    }
    return CRK_OK;
}

// ---------------------------------------------------------------- skin refresh (NEXT-2)
// positions may have left [0, L) by < skin/2 after unwrapped drifts: wrap them (exact)
__global__ void k_wrap(int64_t n, float* x, float* y, float* z, float Lx, float Ly, float Lz) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* c[3] = {x, y, z};
    const float L[3] = {Lx, Ly, Lz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float v = c[a][i];
        if (v >= L[a]) c[a][i] = v - L[a];
        else if (v < 0.f) c[a][i] = v + L[a];
    }
}

__global__ void k_repack(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                         const float* __restrict__ z, const float* __restrict__ m, float4* xm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) xm[i] = make_float4(x[i], y[i], z[i], m[i]);
}

__global__ void k_repack_gas(int64_t ng, const int32_t* __restrict__ gas_idx, const float4* __restrict__ xm,
                             const float* __restrict__ H, float4* gpos) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const int32_t i = gas_idx[g];
    const float4 p = xm[i];
    gpos[g] = make_float4(p.x, p.y, p.z, H[i]);
}

// gravity entry masks of the list's rows (after the fill and after crk_refresh); one warp per row.
// Latency-bound (row start -> records -> boxes): few registers for many resident warps (the
// next entry's record and box requested while the current one is tested); the 8 group boxes in shared memory as packed pairs (groups 2t, 2t + 1),
// two groups per packed-FP32 test.
__global__ void __launch_bounds__(256, 5) k_entry_masks(int64_t na, const int32_t* __restrict__ rowoff,
                                                        const int32_t* __restrict__ rowend, const int2* __restrict__ erec,
                                                        const float4* __restrict__ box8, const int32_t* __restrict__ ifirst,
                                                        const int32_t* __restrict__ icount, const float4* __restrict__ xm,
                                                        float Lx, float Ly, float Lz, float wcut, bool partial, float inv_q,
                                                        int cs, int3 dlo3, int3 dhi3, uint8_t* __restrict__ gmask) {
    __shared__ float s_gb[8][8][6];
    __shared__ float4 s_b[8][4][3];  // [warp][t][axis]: (lo, lo, -hi, -hi) of groups (2t, 2t + 1)
    __shared__ float4 s_off[27];     // periodic offset of each shift code
    const int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < 27) {
        const int code = threadIdx.x;
        s_off[code] = make_float4((float)(code % 3 - 1) * Lx, (float)((code / 3) % 3 - 1) * Ly, (float)(code / 9 - 1) * Lz, 0.f);
    }
    __syncthreads();
    if (a >= na) return;
    const int f0 = ifirst[a], cnt = icount[a];
    const int p0 = rowoff[a], pend = rowend[a];
    // two-stage prefetch: the record two iterations ahead, the box of the next entry (whose record
    // landed an iteration ago) — the record -> box dependency is off the loop's critical path
    auto rec = [&](int q) { return q < pend ? erec[q] : make_int2(0, 0); };
    int2 r = rec(p0 + lane), rn = rec(p0 + lane + 32);
    float4 bl = box8[2 * (int64_t)(r.y & 0x03ffffff)], bh = box8[2 * (int64_t)(r.y & 0x03ffffff) + 1];
    group_boxes(xm, f0, cnt, s_gb[w], lane);  // empty groups: lo = +inf, hi = -inf (never in reach)
    if (lane < 12) {
        const int d = lane / 4, t = lane % 4;
        s_b[w][t][d] = make_float4(s_gb[w][2 * t][d], s_gb[w][2 * t + 1][d], -s_gb[w][2 * t][3 + d], -s_gb[w][2 * t + 1][3 + d]);
    }
    __syncwarp();
    const int dlo[3] = {dlo3.x, dlo3.y, dlo3.z}, dhi[3] = {dhi3.x, dhi3.y, dhi3.z};
    // re-read per test (volatile asm) instead of 24 loop-invariant registers: the kernel wants many warps
    const uint32_t sb = smem_u32(s_b[w]);
    for (int q = p0 + lane; q < pend; q += 32) {
        const int2 rc = r;
        const float4 lc = bl, hc = bh;
        const int2 rnn = rec(q + 64);
        bl = box8[2 * (int64_t)(rn.y & 0x03ffffff)];
        bh = box8[2 * (int64_t)(rn.y & 0x03ffffff) + 1];
        r = rn;
        rn = rnn;
        const float4 of = s_off[(unsigned)rc.y >> 26];
        const float lo[3] = {lc.x + of.x, lc.y + of.y, lc.z + of.z};  // exact (O1)
        const float hi[3] = {hc.x + of.x, hc.y + of.y, hc.z + of.z};
        uint32_t m = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float2 g[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                float4 gb;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(gb.x), "=f"(gb.y), "=f"(gb.z), "=f"(gb.w)
                             : "r"(sb + 16u * (3 * t + d)));
                const float2 u1 = __fadd2_rn(make_float2(lo[d], lo[d]), make_float2(gb.z, gb.w));    // lo_j - hi_g
                const float2 u2 = __fadd2_rn(make_float2(gb.x, gb.y), make_float2(-hi[d], -hi[d]));  // lo_g - hi_j
                g[d] = make_float2(fmaxf(fmaxf(u1.x, u2.x), 0.f), fmaxf(fmaxf(u1.y, u2.y), 0.f));
            }
            const float2 d2 = __ffma2_rn(g[2], g[2], __ffma2_rn(g[1], g[1], __fmul2_rn(g[0], g[0])));
            m |= ((d2.x < wcut ? 1u : 0u) | (d2.y < wcut ? 2u : 0u)) << (2 * t);
        }
        // Newton-3: group g pairs with the leaf only if the leaf reaches past its first particle
        // (16 g < first + count - f0), unless the leaf is a ghost
        const int jend = (rc.x & 0x1fffffff) + ((unsigned)rc.x >> 29) + 1 - f0;
        const int ngr = jend <= 0 ? 0 : min(8, (jend + 15) >> 4);
        if (!(partial && leaf_ghost(lc, hc, inv_q, cs, dlo, dhi))) m &= (1u << ngr) - 1u;
        gmask[q] = (uint8_t)m;
    }
}

crk_status entry_masks(crk_ctx* c, cudaStream_t st) {
    if (c->nleaf[0] <= 0 || !want_masks(c)) return CRK_OK;
    const Layout& L = c->lay;
    k_entry_masks<<<nblk(c->nleaf[0] * 32, 256), 256, 0, st>>>(
        c->nleaf[0], P<int32_t>(c->rowoff[0]), P<int32_t>(c->rowend[0]), P<int2>(c->erec[0]), P<float4>(c->lbox8[1]),
        P<int32_t>(c->lfirst[0]), P<int32_t>(c->lcount[0]), P<float4>(c->xm), L.L[0], L.L[1], L.L[2],
        c->prm.rcut2 * CULL_SLACK, L.partial, L.inv_q, L.cs, make_int3(L.dlo[0], L.dlo[1], L.dlo[2]),
        make_int3(L.dhi[0], L.dhi[1], L.dhi[2]), P<uint8_t>(c->gmask));
    CRK_LAUNCHED(c, "entry masks");
    return CRK_OK;
}

crk_status refresh(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    volatile float* host = reinterpret_cast<float*>(P<char>(c->pinned) + 192);
    Readback rb;
    rb.add(P<float>(c->disp) + 1, 192, 4);
    CRK_TRY(readback(c, rb, st));
    CRK_TRY(cuda_check(c, cudaStreamSynchronize(st), "sync"));
    if (!(*host < 0.5f * c->prm.skin)) {
        c->skin_lists = false;
        return fail(c, CRK_ESTATE, "the displacement since the build reached skin/2: call crk_build_lists");
    }
    const int64_t n = c->n;
    k_repack<<<nblk(n, 256), 256, 0, st>>>(n, p->x, p->y, p->z, p->m, P<float4>(c->xm));
    CRK_LAUNCHED(c, "repack");
    if (c->n_gas > 0) {
        k_repack_gas<<<nblk(c->n_gas, 256), 256, 0, st>>>(c->n_gas, P<int32_t>(c->gas_idx), P<float4>(c->xm), p->H,
                                                           P<float4>(c->gpos));
        CRK_LAUNCHED(c, "repack gas");
    }
    for (int s = 0; s < 4; ++s) CRK_TRY(leaf_boxes(c, s, st));
    CRK_TRY(entry_masks(c, st));
    c->stage = ST_LISTS;  // the displacement bound keeps accumulating until the next build
    return CRK_OK;
}

crk_status build_lists(crk_ctx* c, crk_particles* p, cudaStream_t st) {
    const int64_t n = p->n;
    const Layout& L = c->lay;
    c->n = n;
    c->stage = ST_NONE;
    const int bits = 3 * (L.cbits + L.fbits);
    // ---- buffers
    CRK_TRY(grow(c, c->keys_a, n * 4, st));
    CRK_TRY(grow(c, c->keys_b, n * 4, st));
    CRK_TRY(grow(c, c->idx_a, n * 4, st));
    CRK_TRY(grow(c, c->idx_b, n * 4, st));
    CRK_TRY(grow(c, c->scratch, n * 48 + 64, st));
    CRK_TRY(grow(c, c->xm, (n + JMAX) * 16, st));  // + one j-leaf of padding: whole-leaf reads
    CRK_TRY(grow(c, c->gflag, (n + 1) * 4, st));
    CRK_TRY(grow(c, c->grank, (n + 1) * 4, st));
    CRK_TRY(grow(c, c->cell_start, L.ncm * 4, st));
    CRK_TRY(grow(c, c->cell_end, L.ncm * 4, st));
    CRK_TRY(grow(c, c->leaf_cnt, 4 * (L.ncm + 1) * 4, st));
    CRK_TRY(grow(c, c->dev_scalars, 64, st));
    CRK_TRY(grow(c, c->gas_idx, n * 4, st));
    CRK_TRY(grow(c, c->gpos, n * 16, st));
    if (n == 0) return fail(c, CRK_EINVAL, "no particles");
    if (c->prm.skin > 0.f) {  // positions may lie outside the box by < skin/2 after unwrapped drifts
        k_wrap<<<nblk(n, 256), 256, 0, st>>>(n, p->x, p->y, p->z, L.L[0], L.L[1], L.L[2]);
        CRK_LAUNCHED(c, "wrap");
    }

    // ---- keys + sort (32-bit keys, 3 (cbits + fbits) significant bits)
    SoA in;
    float* f32[9] = {p->x, p->y, p->z, p->vx, p->vy, p->vz, p->m, p->H, p->u};
    for (int t = 0; t < 9; ++t) in.f[t] = f32[t];
    in.sp = p->species;
    in.id = p->id;
    float4* rec = P<float4>(c->scratch);
    // counting sort by cell, then a segmented sort of every cell by its in-cell key (the leaf-count
    // buffer, written later, holds the cell histogram and offsets meanwhile)
    int32_t* ccount = P<int32_t>(c->leaf_cnt);
    int32_t* coff = ccount + (L.ncm + 1);
    CRK_TRY(cuda_check(c, zero_async(ccount, (L.ncm + 1) * 4, st, c), "memset"));
    k_keys<<<nblk(n, 256), 256, 0, st>>>(n, in, L.inv_q, L.cs, L.fbits, P<uint32_t>(c->keys_a), P<int32_t>(c->idx_a),
                                         rec, ccount);
    CRK_LAUNCHED(c, "keys");
    size_t tmp = 0;
    cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, P<uint32_t>(c->keys_b), P<uint32_t>(c->keys_a),
                                        P<int32_t>(c->idx_b), P<int32_t>(c->idx_a), (int)n, (int)L.ncm, coff, coff + 1,
                                        st);
    size_t tmp2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp2, P<int32_t>(c->gflag), P<int32_t>(c->grank), (int)(n + 1), st);
    size_t tmp3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp3, P<int32_t>(c->leaf_cnt), P<int32_t>(c->leaf_cnt), (int)(L.ncm + 1), st);
    size_t need = tmp > tmp2 ? tmp : tmp2;
    need = need > tmp3 ? need : tmp3;
    need = need > (size_t)(n + 1) * 4 ? need : (size_t)(n + 1) * 4;
    CRK_TRY(grow(c, c->cub_tmp, need, st));
    tmp = c->cub_tmp.cap;
    CRK_TRY(cuda_check(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, ccount, coff, (int)(L.ncm + 1), st),
                       "cell scan"));
    c->launches += 2;
    CRK_TRY(cuda_check(c, zero_async(c->cell_end.p, L.ncm * 4, st, c), "memset"));  // the scatter's cursors
    k_cell_scatter<<<nblk(n, 256), 256, 0, st>>>(n, P<uint32_t>(c->keys_a), L.fbits, coff, P<int32_t>(c->cell_end),
                                                 P<uint32_t>(c->keys_b), P<int32_t>(c->idx_b));
    CRK_LAUNCHED(c, "cell scatter");
    // cells up to CELL_SORT_MAX particles: one warp each (radix by the in-cell bits); larger ones
    // (clustered inputs): CUB's segmented
    // sort over (beg, end) segments, empty for the small cells
    int32_t* beg = ccount;  // the histogram is consumed
    int32_t* end = ccount + 2 * (L.ncm + 1);
    CRK_TRY(grow(c, c->work, 64, st));
    int* nbig = P<int>(c->work) + 12;
    CRK_TRY(cuda_check(c, zero_async(nbig, 4, st, c), "memset"));
    k_cell_sort<<<nblk(L.ncm, 8), 256, 0, st>>>(L.ncm, 3 * L.fbits, coff, P<uint32_t>(c->keys_b), P<int32_t>(c->idx_b),
                                                P<uint32_t>(c->keys_a), P<int32_t>(c->idx_a), beg, end, nbig);
    CRK_LAUNCHED(c, "cell sort");
    {  // CUB's segmented sort only when some cell is large: it reads partition sizes back with a
       // copy-engine transfer, which would queue behind the caller's bulk copies
        Readback rb;
        rb.add(nbig, 64, 4);
        CRK_TRY(readback(c, rb, st));
        CRK_TRY(cuda_check(c, cudaStreamSynchronize(st), "sync"));
        if (reinterpret_cast<volatile int32_t*>(P<char>(c->pinned))[16] > 0) {
            tmp = c->cub_tmp.cap;
            CRK_TRY(cuda_check(c, cub::DeviceSegmentedSort::SortPairs(c->cub_tmp.p, tmp, P<uint32_t>(c->keys_b),
                                                                      P<uint32_t>(c->keys_a), P<int32_t>(c->idx_b),
                                                                      P<int32_t>(c->idx_a), (int)n, (int)L.ncm, beg,
                                                                      end, st), "segmented sort (large cells)"));
            c->launches += 3;
        }
    }
    (void)bits;
    const uint32_t* keys = P<uint32_t>(c->keys_a);
    int32_t* perm = P<int32_t>(c->idx_a);
    k_tie_fix<<<nblk(n, 256), 256, 0, st>>>(n, keys, perm, p->id);
    CRK_LAUNCHED(c, "tie fix");

    // ---- permute the caller's arrays in place: one gather of the packed records
    CRK_TRY(cuda_check(c, zero_async(c->cell_start.p, L.ncm * 4, st, c), "memset"));
    CRK_TRY(cuda_check(c, zero_async(c->cell_end.p, L.ncm * 4, st, c), "memset"));
    CRK_TRY(cuda_check(c, zero_async(P<int32_t>(c->gflag) + n, 4, st, c), "memset"));
    CRK_TRY(cuda_check(c, zero_async(c->dev_scalars.p, 64, st, c), "memset"));
    k_permute<<<nblk(n, 256), 256, 0, st>>>(n, perm, rec, in, keys, L.fbits, P<float4>(c->xm), P<int32_t>(c->gflag),
                                            P<int32_t>(c->cell_start), P<int32_t>(c->cell_end), p->perm);
    CRK_LAUNCHED(c, "permute");

    // ---- gas ranks
    tmp = c->cub_tmp.cap;
    CRK_TRY(cuda_check(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, P<int32_t>(c->gflag), P<int32_t>(c->grank),
                                                        (int)(n + 1), st), "gas scan"));
    c->launches += 2;
    k_gas_pack<<<nblk(n, 256), 256, 0, st>>>(n, P<int32_t>(c->gflag), P<int32_t>(c->grank), P<float4>(c->xm), p->H,
                                             P<int32_t>(c->gas_idx), P<float4>(c->gpos), P<float>(c->dev_scalars));
    CRK_LAUNCHED(c, "gas pack");

    // ---- leaves
    const int lmax[4] = {c->prm.leaf_max_i, c->prm.leaf_max_j, c->prm.leaf_max_gas_i, c->prm.leaf_max_gas_j};
    int32_t* cnt = P<int32_t>(c->leaf_cnt);
    Dom dom;
    for (int d = 0; d < 3; ++d) { dom.lo[d] = L.dlo[d]; dom.hi[d] = L.dhi[d]; }
    k_leaf_counts<<<nblk(L.ncm + 1, 256), 256, 0, st>>>(L.ncm, P<int32_t>(c->cell_start), P<int32_t>(c->cell_end),
                                                        P<int32_t>(c->grank), lmax[0], lmax[1], lmax[2], lmax[3], dom,
                                                        cnt);
    CRK_LAUNCHED(c, "leaf counts");
    for (int s = 0; s < 4; ++s) {
        tmp = c->cub_tmp.cap;
        CRK_TRY(cuda_check(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, cnt + s * (L.ncm + 1),
                                                            cnt + s * (L.ncm + 1), (int)(L.ncm + 1), st), "leaf scan"));
        c->launches += 2;
    }
    // totals: leaf counts (4) + n_gas, one synchronisation
    volatile int32_t* host = P<int32_t>(c->pinned);
    {
        Readback rb;
        for (int s = 0; s < 4; ++s) rb.add(cnt + s * (L.ncm + 1) + L.ncm, 4 * s, 4);
        rb.add(P<int32_t>(c->grank) + n, 16, 4);
        rb.add(P<int32_t>(c->dev_scalars), 20, 4);  // max fl32(H^2) over gas (k_gas_pack), float bits
        CRK_TRY(readback(c, rb, st));
    }
    CRK_TRY(cuda_check(c, cudaStreamSynchronize(st), "sync"));
    for (int s = 0; s < 4; ++s) c->nleaf[s] = host[s];
    c->n_gas = host[4];
    {
        // packed list entries keep the j-leaf index in 26 bits (leaf | shift << 26)
        if (c->nleaf[1] >= (1 << 26) || c->nleaf[3] >= (1 << 26))
            return fail(c, CRK_ECAPACITY, "more than 2^26 - 1 j-leaves (packed list entries)");
        // H < box/4 (as r_c): the minimum-image and one-shift list search assume it
        const int32_t hb = host[5];
        float h2max;
        memcpy(&h2max, &hb, 4);
        for (int a = 0; a < 3; ++a)
            if (!(std::sqrt((double)h2max) < c->prm.box[a] / 4))
                return fail(c, CRK_EINVAL, "every gas H must be < box/4");
    }
    for (int s = 0; s < 4; ++s) {
        const int64_t nl = c->nleaf[s] > 0 ? c->nleaf[s] : 1;
        CRK_TRY(grow(c, c->lfirst[s], nl * 4, st));
        CRK_TRY(grow(c, c->lcount[s], nl * 4, st));
        CRK_TRY(grow(c, c->lbbox[s], nl * 24, st));
        CRK_TRY(grow(c, c->lcell[s], nl * 8, st));
        CRK_TRY(grow(c, c->lbox8[s], nl * 32, st));
        if (s >= 2) CRK_TRY(grow(c, c->lmaxh2[s], nl * 4, st));
        k_leaf_fill<<<nblk(L.ncm, 256), 256, 0, st>>>(L.ncm, P<int32_t>(c->cell_start), P<int32_t>(c->cell_end),
                                                      P<int32_t>(c->grank), cnt + s * (L.ncm + 1), s, lmax[s],
                                                      dom, P<int32_t>(c->lfirst[s]), P<int32_t>(c->lcount[s]),
                                                      P<uint64_t>(c->lcell[s]));
        CRK_LAUNCHED(c, "leaf fill");
        CRK_TRY(leaf_boxes(c, s, st));
    }

    // ---- lists: count, scan, fill
    Readback rbl;
    for (int m = 0; m < 2; ++m) {
        const int64_t na = c->nleaf[m == 0 ? 0 : 2];
        CRK_TRY(grow(c, c->rowlen[m], (na + 1) * 4, st));
        CRK_TRY(grow(c, c->rowoff[m], (na + 1) * 4, st));
        CRK_TRY(grow(c, c->rowend[m], (na + 1) * 4, st));
        ListArgs A = list_args(c, m);
        CRK_TRY(cuda_check(c, zero_async(P<int32_t>(c->rowlen[m]) + na, 4, st, c), "memset"));
        if (na > 0) {
            k_lists<false><<<nblk(na * 32, LIST_WARPS * 32), LIST_WARPS * 32, 0, st>>>(A);
            CRK_LAUNCHED(c, "list bound");
        }
        tmp = c->cub_tmp.cap;
        CRK_TRY(cuda_check(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, P<int32_t>(c->rowlen[m]),
                                                            P<int32_t>(c->rowoff[m]), (int)(na + 1), st), "row scan"));
        c->launches += 2;
        rbl.add(P<int32_t>(c->rowoff[m]) + na, 4 * (8 + m), 4);
    }
    CRK_TRY(readback(c, rbl, st));
    CRK_TRY(cuda_check(c, cudaStreamSynchronize(st), "sync"));
    for (int m = 0; m < 2; ++m) {
        c->nent[m] = host[8 + m];
        const int64_t na = c->nleaf[m == 0 ? 0 : 2];
        const int64_t ne = c->nent[m] > 0 ? c->nent[m] : 1;
        CRK_TRY(grow(c, c->erec[m], ne * 8, st));
        if (m == 0) CRK_TRY(grow(c, c->gmask, ne + 256, st));
        if (m == 1) {  // row classes (interior / holds ghosts) for crk_select_rows; all interior when whole
            CRK_TRY(grow(c, c->rclass, na + 16, st));
            if (!L.partial) CRK_TRY(cuda_check(c, zero_async(c->rclass.p, na + 16, st, c), "memset"));
        }
        ListArgs A = list_args(c, m);
        if (na > 0) {
            k_lists<true><<<nblk(na * 32, LIST_WARPS * 32), LIST_WARPS * 32, 0, st>>>(A);
            CRK_LAUNCHED(c, "list fill");
        }
    }
    CRK_TRY(entry_masks(c, st));
    // ---- gas-ordered state buffers for the hydro passes
    const int64_t ng = c->n_gas > 0 ? c->n_gas : 1;
    CRK_TRY(grow(c, c->gvel, ng * 16, st));
    CRK_TRY(grow(c, c->gV, ng * 4, st));
    CRK_TRY(grow(c, c->gposV, ng * 16, st));
    CRK_TRY(grow(c, c->gcoef, ng * 16 * 4, st));
    CRK_TRY(grow(c, c->grec, ng * 9 * 16, st));
    CRK_TRY(grow(c, c->gu, ng * 4, st));
    // scratch of the later passes sized here, in stream order, so that gravity (a3) and
    // geometry (a4) may run concurrently on two streams without either reallocating
    CRK_TRY(grow(c, c->gacc, (n > ng ? n : ng) * 16, st));
    CRK_TRY(grow(c, c->work, 64, st));
    if (c->nbr_cap > 0) {
        CRK_TRY(grow(c, c->nbr, (size_t)ng * c->nbr_cap * sizeof(uint16_t), st));
        CRK_TRY(grow(c, c->ncnt, (size_t)ng * sizeof(int32_t) + 64, st));  // + pad: 16-byte-aligned bulk reads
        CRK_TRY(grow(c, c->lflag, (size_t)(2 * c->nleaf[2] + 1) * sizeof(int32_t), st));
    }
    if (c->prm.skin > 0.f) {
        CRK_TRY(grow(c, c->disp, 16, st));
        CRK_TRY(cuda_check(c, zero_async(c->disp.p, 16, st, c), "memset"));
    }
    c->skin_lists = c->prm.skin > 0.f;
    c->csr_views = false;
    c->row_sel = 0;
    c->stage = ST_LISTS;
    return CRK_OK;
}

// crk_list_view's CSR (compacted: rows are stored at their bounds) col / shift arrays, decoded
// from the packed entries, one warp per row
__global__ void k_decode_rows(int64_t na, const int32_t* __restrict__ rowoff, const int32_t* __restrict__ rowend,
                              const int32_t* __restrict__ csroff, const int2* __restrict__ erec, int32_t* col,
                              int8_t* shift) {
    const int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (a >= na) return;
    const int lane = threadIdx.x & 31;
    const int b0 = rowoff[a], b1 = rowend[a], o = csroff[a];
    for (int p = b0 + lane; p < b1; p += 32) {
        const int2 r = erec[p];
        col[o + p - b0] = r.y & 0x03ffffff;
        shift[o + p - b0] = (int8_t)((unsigned)r.y >> 26);
    }
}

__global__ void k_row_lengths(int64_t na, const int32_t* __restrict__ rowoff, const int32_t* __restrict__ rowend,
                              int32_t* len) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a < na) len[a] = rowend[a] - rowoff[a];
    if (a == na) len[a] = 0;
}

crk_status csr_views(crk_ctx* c) {
    if (c->csr_views) return CRK_OK;
    for (int m = 0; m < 2; ++m) {
        const int64_t na = c->nleaf[m == 0 ? 0 : 2];
        CRK_TRY(grow(c, c->csroff[m], (na + 1) * 4, 0));
        k_row_lengths<<<nblk(na + 1, 256), 256>>>(na, P<int32_t>(c->rowoff[m]), P<int32_t>(c->rowend[m]),
                                                  P<int32_t>(c->rowlen[m]));
        CRK_LAUNCHED(c, "row lengths");
        size_t tmp = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp, P<int32_t>(c->rowlen[m]), P<int32_t>(c->csroff[m]), (int)(na + 1));
        CRK_TRY(grow(c, c->cub_tmp, tmp, 0));
        tmp = c->cub_tmp.cap;
        CRK_TRY(cuda_check(c, cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, P<int32_t>(c->rowlen[m]),
                                                            P<int32_t>(c->csroff[m]), (int)(na + 1)), "csr scan"));
        c->launches += 2;
        int32_t tot = 0;
        CRK_TRY(cuda_check(c, cudaMemcpy(&tot, P<int32_t>(c->csroff[m]) + na, 4, cudaMemcpyDeviceToHost), "csr size"));
        c->nlist[m] = tot;
        CRK_TRY(grow(c, c->col[m], (size_t)(tot > 0 ? tot : 1) * 4, 0));
        CRK_TRY(grow(c, c->shift[m], (size_t)(tot > 0 ? tot : 1), 0));
        if (na > 0) {
            k_decode_rows<<<nblk(na * 32, 256), 256>>>(na, P<int32_t>(c->rowoff[m]), P<int32_t>(c->rowend[m]),
                                                       P<int32_t>(c->csroff[m]), P<int2>(c->erec[m]),
                                                       P<int32_t>(c->col[m]), P<int8_t>(c->shift[m]));
            CRK_LAUNCHED(c, "decode entries");
        }
    }
    CRK_TRY(cuda_check(c, cudaDeviceSynchronize(), "sync"));
    c->csr_views = true;
    return CRK_OK;
}

}  // namespace crk
