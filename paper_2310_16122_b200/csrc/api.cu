// api.cu — the extern "C" boundary of libcrksr.so (include/crksr.h): context lifetime,
// parameter validation, call-order state machine, error reporting.
#include <cmath>
#include <cstring>
#include <new>


#include "common.cuh"

namespace crk {

crk_status build_lists(crk_ctx* c, crk_particles* p, cudaStream_t st);
crk_status gravity_kick(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st);
crk_status gravity_count(crk_ctx* c, crk_particles* p, int32_t* cnt, cudaStream_t st);
crk_status geometry(crk_ctx* c, crk_particles* p, cudaStream_t st);
crk_status corrections(crk_ctx* c, crk_particles* p, cudaStream_t st);
crk_status extras(crk_ctx* c, crk_particles* p, cudaStream_t st);
crk_status corrections_extras(crk_ctx* c, crk_particles* p, cudaStream_t st);
crk_status csr_views(crk_ctx* c);
crk_status update_h(crk_ctx* c, int kth, float factor, float* H_out, int32_t* n_unconverged, cudaStream_t st);
crk_status accel_dudt(crk_ctx* c, crk_particles* p, float dt, cudaStream_t st);
crk_status hydro_count(crk_ctx* c, int32_t* cgather, int32_t* csym, cudaStream_t st);
crk_status neighbour_lists(crk_ctx* c, int32_t cap_out, int32_t* count, int32_t* nbr, cudaStream_t st);

crk_status fail(crk_ctx* c, crk_status s, const char* what) {
    if (c) c->err = what;
    return s;
}

crk_status cuda_check(crk_ctx* c, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return CRK_OK;
    if (c) c->err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? CRK_ENOMEM : CRK_ECUDA;
}

__global__ void k_readback(Readback r, char* dst) {
    for (int i = 0; i < r.n; ++i) {
        if (r.bytes[i] == 8)
            *reinterpret_cast<volatile int64_t*>(dst + r.dst[i]) = *reinterpret_cast<const int64_t*>(r.src[i]);
        else
            *reinterpret_cast<volatile int32_t*>(dst + r.dst[i]) = *reinterpret_cast<const int32_t*>(r.src[i]);
    }
    __threadfence_system();
}

__global__ void k_zero(uint4* p16, size_t n16, char* tail, int ntail) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t k = i; k < n16; k += stride) p16[k] = make_uint4(0u, 0u, 0u, 0u);
    if (i < (size_t)ntail) tail[i] = 0;
}

cudaError_t zero_async(void* p, size_t bytes, cudaStream_t st, crk_ctx* c) {
    if (bytes == 0) return cudaSuccess;
    char* b = static_cast<char*>(p);
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(b) & 15)) & 15;  // unaligned prefix bytes
    const size_t pre = head < bytes ? head : bytes;
    const size_t n16 = (bytes - pre) / 16;
    const size_t rest = bytes - pre - 16 * n16;
    // prefix and suffix (< 16 bytes each) by a second tiny launch
    if (pre) {
        k_zero<<<1, 32, 0, st>>>(nullptr, 0, b, (int)pre);
        if (c) c->launches++;
    }
    if (n16 || rest) {
        if (c) c->launches++;
        const size_t blocks = n16 ? (n16 + 255) / 256 : 1;
        k_zero<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(reinterpret_cast<uint4*>(b + pre), n16,
                                                                        b + pre + 16 * n16, (int)rest);
    }
    return cudaGetLastError();
}

crk_status readback(crk_ctx* c, const Readback& r, cudaStream_t st) {
    k_readback<<<1, 1, 0, st>>>(r, static_cast<char*>(c->pinned_dev));
    CRK_LAUNCHED(c, "readback");
    return CRK_OK;
}

crk_status grow(crk_ctx* c, Buf& b, size_t bytes, cudaStream_t st) {
    if (bytes <= b.cap) return CRK_OK;
    if (b.p) {
        cudaError_t e = cudaFreeAsync(b.p, st);
        if (e != cudaSuccess) return cuda_check(c, e, "cudaFreeAsync");
        b.p = nullptr;
        b.cap = 0;
    }
    size_t want = bytes + bytes / 8 + 256;
    cudaError_t e = cudaMallocAsync(&b.p, want, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_check(c, e, "cudaMallocAsync");
    }
    b.cap = want;
    return CRK_OK;
}

static bool pow2(double v) {
    if (!(v > 0)) return false;
    int e;
    return std::frexp(v, &e) == 0.5;
}

static crk_status validate(const crk_params* p, Layout& L, std::string& why) {
    double lmax = 0;
    for (int a = 0; a < 3; ++a) {
        if (!pow2(p->box[a]) || p->box[a] < 16 || p->box[a] > 4096) { why = "box must be powers of two in [16, 4096]"; return CRK_EINVAL; }
        lmax = p->box[a] > lmax ? p->box[a] : lmax;
    }
    if (!pow2(p->cell_side) || p->cell_side < 1.0) { why = "cell_side must be a power of two >= 1"; return CRK_EINVAL; }
    for (int a = 0; a < 3; ++a)
        if (p->cell_side > p->box[a] / 4) { why = "cell_side must be <= box/4"; return CRK_EINVAL; }
    for (int a = 0; a < 3; ++a)
        if (!(p->rcut2 > 0) || std::sqrt((double)p->rcut2) >= p->box[a] / 4) { why = "need 0 < rcut < box/4"; return CRK_EINVAL; }
    if (!(p->eps2 > 0)) { why = "eps2 must be > 0"; return CRK_EINVAL; }
    if (!(p->leaf_max_i == 16 || p->leaf_max_i == 32 || p->leaf_max_i == 64 || p->leaf_max_i == 128) ||
        p->leaf_max_i > GRAV_NW * GRAV_G) { why = "leaf_max_i must be 16, 32, 64 or 128"; return CRK_EINVAL; }
    if (p->leaf_max_j != JMAX || p->leaf_max_gas_j != JMAX) { why = "leaf_max_j and leaf_max_gas_j must be 8"; return CRK_EINVAL; }
    if (!(p->leaf_max_gas_i == 16 || p->leaf_max_gas_i == 32 || p->leaf_max_gas_i == 64) ||
        p->leaf_max_gas_i > HYD_NW * HYD_G) { why = "leaf_max_gas_i must be 16, 32 or 64"; return CRK_EINVAL; }
    if (!(p->gamma > 1.f)) { why = "gamma must be > 1"; return CRK_EINVAL; }
    L.q = std::ldexp(lmax, -23);
    L.inv_q = (float)(1.0 / L.q);
    L.cs = (int)std::lround(std::log2(p->cell_side / L.q));
    int maxn = 1;
    for (int a = 0; a < 3; ++a) {
        L.ncell[a] = (int)std::lround(p->box[a] / p->cell_side);
        maxn = L.ncell[a] > maxn ? L.ncell[a] : maxn;
        L.L[a] = (float)p->box[a];
    }
    if (maxn > 256) { why = "at most 256 cells per axis (raise cell_side)"; return CRK_EINVAL; }
    L.cbits = 0;
    while ((1 << L.cbits) < maxn) ++L.cbits;
    L.fbits = (32 - 3 * L.cbits) / 3;  // 32-bit sort keys (DESIGN.md §2 O3)
    if (L.fbits > L.cs) L.fbits = L.cs;
    L.ncm = (int64_t)1 << (3 * L.cbits);
    bool whole = p->dom_hi[0] == 0 && p->dom_hi[1] == 0 && p->dom_hi[2] == 0;
    L.partial = false;
    for (int a = 0; a < 3; ++a) {
        L.dlo[a] = whole ? 0 : p->dom_lo[a];
        L.dhi[a] = whole ? L.ncell[a] : p->dom_hi[a];
        if (L.dlo[a] < 0 || L.dhi[a] > L.ncell[a] || L.dlo[a] >= L.dhi[a]) { why = "bad domain cell range"; return CRK_EINVAL; }
        if (L.dlo[a] != 0 || L.dhi[a] != L.ncell[a]) L.partial = true;
    }
    if (!(p->skin >= 0.f) || p->skin >= p->cell_side) { why = "skin must be in [0, cell_side)"; return CRK_EINVAL; }
    if (p->skin > 0.f && L.partial) { why = "a skin needs a whole-box domain"; return CRK_EINVAL; }
    if (!((p->grav_kernel >= 0 && p->grav_kernel <= 2) || (p->grav_kernel >= 6 && p->grav_kernel <= 8))) {
        why = "grav_kernel must be 0-2 or 6-8"; return CRK_EINVAL;
    }
    if (!(p->hydro_kernel == 0 || p->hydro_kernel == 2 || (p->hydro_kernel >= 4 && p->hydro_kernel <= 6))) {
        why = "hydro_kernel must be 0, 2, 4, 5 or 6"; return CRK_EINVAL;
    }
    if (p->nbr_cap > 65535) { why = "nbr_cap must be <= 65535"; return CRK_EINVAL; }
    return CRK_OK;
}

}  // namespace crk

using namespace crk;

extern "C" {

crk_status crk_create(const crk_params* params, int device, crk_ctx** out) {
    if (!params || !out) return CRK_EINVAL;
    *out = nullptr;
    Layout L;
    std::string why;
    crk_status s = validate(params, L, why);
    if (s != CRK_OK) return s;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return CRK_ECUDA;
    crk_ctx* c = new (std::nothrow) crk_ctx();
    if (!c) return CRK_ENOMEM;
    c->prm = *params;
    c->device = device;
    c->lay = L;
    void* h = nullptr;
    e = cudaHostAlloc(&h, 256, cudaHostAllocMapped);
    if (e != cudaSuccess) {
        delete c;
        return CRK_ENOMEM;
    }
    c->pinned.p = h;
    c->pinned.cap = 256;
    if (cudaHostGetDevicePointer(&c->pinned_dev, h, 0) != cudaSuccess) {
        cudaFreeHost(h);
        delete c;
        return CRK_ECUDA;
    }
    // gas neighbour-list capacity per particle (crk_params.nbr_cap: 0 = default, < 0 = off)
    c->nbr_cap = params->nbr_cap == 0 ? 128 : (params->nbr_cap < 0 ? 0 : params->nbr_cap);
    // the gravity kernel's dynamic shared memory fits in the default 48 KB
    *out = c;
    return CRK_OK;
}

crk_status crk_destroy(crk_ctx* c) {
    if (!c) return CRK_EINVAL;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    Buf* bufs[] = {&c->keys_a, &c->keys_b, &c->idx_a, &c->idx_b, &c->cub_tmp, &c->scratch, &c->xm,
                   &c->cell_start, &c->cell_end, &c->leaf_cnt, &c->gflag, &c->grank, &c->gas_idx,
                   &c->dev_scalars, &c->gpos, &c->gvel, &c->gV, &c->gcoef, &c->grec, &c->gu,
                   &c->gacc, &c->gposV, &c->sel_flag, &c->sel_mask, &c->work, &c->nbr, &c->ncnt, &c->lflag, &c->gmask, &c->rclass, &c->disp};
    for (Buf* b : bufs)
        if (b->p) cudaFree(b->p);
    for (int s = 0; s < 4; ++s) {
        Buf* lb[] = {&c->lfirst[s], &c->lcount[s], &c->lbbox[s], &c->lmaxh2[s], &c->lcell[s], &c->lbox8[s]};
        for (Buf* b : lb)
            if (b->p) cudaFree(b->p);
    }
    for (int m = 0; m < 2; ++m) {
        Buf* lb[] = {&c->rowlen[m], &c->rowoff[m], &c->col[m], &c->shift[m], &c->erec[m], &c->rowend[m], &c->csroff[m]};
        for (Buf* b : lb)
            if (b->p) cudaFree(b->p);
    }
    if (c->pinned.p) cudaFreeHost(c->pinned.p);
    delete c;
    return CRK_OK;
}

static crk_status check_parts(crk_ctx* c, const crk_particles* p, bool need_built) {
    if (!c) return CRK_EINVAL;
    if (!p || !p->x || !p->y || !p->z || !p->m || !p->species || !p->id || !p->H || p->n <= 0)
        return fail(c, CRK_EINVAL, "missing particle arrays");
    if (p->n >= ((int64_t)1 << 29)) return fail(c, CRK_EINVAL, "n must be < 2^29 (packed list entries)");
    if (c->prm.symmetric && p->n >= ((int64_t)1 << 30)) return fail(c, CRK_EINVAL, "n too large for symmetric mode");
    if (need_built && (c->stage < ST_LISTS || p->n != c->n)) return fail(c, CRK_ESTATE, "call crk_build_lists first");
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return cuda_check(c, e, "cudaSetDevice");
    return CRK_OK;
}

crk_status crk_build_lists(crk_ctx* c, crk_particles* p, void* stream) {
    CRK_TRY(check_parts(c, p, false));
    if (!p->vx || !p->vy || !p->vz || !p->u) return fail(c, CRK_EINVAL, "missing particle arrays");
    return build_lists(c, p, (cudaStream_t)stream);
}

crk_status crk_gravity_kick(crk_ctx* c, crk_particles* p, float dt, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    return gravity_kick(c, p, dt, (cudaStream_t)stream);
}

crk_status crk_geometry(crk_ctx* c, crk_particles* p, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    CRK_TRY(geometry(c, p, (cudaStream_t)stream));
    c->stage = ST_GEO;
    return CRK_OK;
}

crk_status crk_corrections(crk_ctx* c, crk_particles* p, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    if (c->stage < ST_GEO) return fail(c, CRK_ESTATE, "call crk_geometry first");
    CRK_TRY(corrections(c, p, (cudaStream_t)stream));
    c->stage = ST_COR;
    return CRK_OK;
}

crk_status crk_extras(crk_ctx* c, crk_particles* p, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    if (c->stage < ST_COR) return fail(c, CRK_ESTATE, "call crk_corrections first");
    if (!p->vx || !p->vy || !p->vz || !p->u) return fail(c, CRK_EINVAL, "extras needs v and u");
    CRK_TRY(extras(c, p, (cudaStream_t)stream));
    c->stage = ST_EXT;
    return CRK_OK;
}

crk_status crk_corrections_extras(crk_ctx* c, crk_particles* p, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    if (c->stage < ST_GEO) return fail(c, CRK_ESTATE, "call crk_geometry first");
    if (!p->vx || !p->vy || !p->vz || !p->u) return fail(c, CRK_EINVAL, "extras needs v and u");
    CRK_TRY(corrections_extras(c, p, (cudaStream_t)stream));
    c->stage = ST_EXT;
    return CRK_OK;
}

crk_status crk_select_rows(crk_ctx* c, int32_t which) {
    if (!c) return CRK_EINVAL;
    if (which < 0 || which > 2) return fail(c, CRK_EINVAL, "which must be 0 (all rows), 1 (interior) or 2 (ghost rows)");
    if (which != 0 && c->stage < ST_LISTS) return fail(c, CRK_ESTATE, "call crk_build_lists first");
    c->row_sel = which;
    return CRK_OK;
}

crk_status crk_update_h(crk_ctx* c, crk_particles* p, int32_t k_ngb, float factor, float* H_out,
                        int32_t* n_unconverged, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    if (c->stage < ST_GEO) return fail(c, CRK_ESTATE, "call crk_geometry first (it builds the neighbour lists)");
    if (k_ngb < 1 || k_ngb > 127 || !(factor > 0.f) || !H_out || !n_unconverged)
        return fail(c, CRK_EINVAL, "k_ngb in [1, 127], factor > 0, H_out and n_unconverged required");
    return update_h(c, k_ngb, factor, H_out, n_unconverged, (cudaStream_t)stream);
}

crk_status crk_hydro_accel_dudt(crk_ctx* c, crk_particles* p, float dt, void* stream) {
    CRK_TRY(check_parts(c, p, true));
    if (c->stage < ST_EXT) return fail(c, CRK_ESTATE, "call crk_extras first");
    return accel_dudt(c, p, dt, (cudaStream_t)stream);
}

crk_status crk_count_pairs(crk_ctx* c, crk_particles* p, int32_t* cgrav, int32_t* cgather, int32_t* csym,
                           void* stream) {
    CRK_TRY(check_parts(c, p, true));
    if (!cgrav || !cgather || !csym) return fail(c, CRK_EINVAL, "null count array");
    cudaStream_t st = (cudaStream_t)stream;
    CRK_TRY(cuda_check(c, zero_async(cgrav, p->n * 4, st, c), "memset"));
    CRK_TRY(cuda_check(c, zero_async(cgather, p->n * 4, st, c), "memset"));
    CRK_TRY(cuda_check(c, zero_async(csym, p->n * 4, st, c), "memset"));
    CRK_TRY(gravity_count(c, p, cgrav, st));
    return hydro_count(c, cgather, csym, st);
}

crk_status crk_neighbour_lists(crk_ctx* c, int32_t cap_out, int32_t* count, int32_t* nbr, void* stream) {
    if (!c) return CRK_EINVAL;
    if (cap_out < 1 || !count || !nbr) return fail(c, CRK_EINVAL, "cap_out >= 1, count and nbr required");
    if (c->nbr_cap <= 0) return fail(c, CRK_ESTATE, "the neighbour lists are off (crk_params.nbr_cap < 0)");
    if (c->stage < ST_GEO) return fail(c, CRK_ESTATE, "call crk_geometry first (it builds the neighbour lists)");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    return neighbour_lists(c, cap_out, count, nbr, (cudaStream_t)stream);
}

crk_status crk_list_view(crk_ctx* c, crk_lists* o) {
    if (!c || !o) return CRK_EINVAL;
    if (c->stage < ST_LISTS) return fail(c, CRK_ESTATE, "call crk_build_lists first");
    CRK_TRY(cuda_check(c, cudaSetDevice(c->device), "cudaSetDevice"));
    CRK_TRY(csr_views(c));
    for (int s = 0; s < 4; ++s) {
        o->n_leaf[s] = c->nleaf[s];
        o->leaf_first[s] = P<int32_t>(c->lfirst[s]);
        o->leaf_count[s] = P<int32_t>(c->lcount[s]);
        o->leaf_bbox[s] = P<float>(c->lbbox[s]);
        o->leaf_maxh2[s] = s >= 2 ? P<float>(c->lmaxh2[s]) : nullptr;
        o->leaf_cell[s] = P<uint64_t>(c->lcell[s]);
    }
    o->n_gas = c->n_gas;
    o->gas_idx = P<int32_t>(c->gas_idx);
    for (int m = 0; m < 2; ++m) {
        o->n_entries[m] = c->nlist[m];
        o->row_off[m] = P<int32_t>(c->csroff[m]);
        o->col[m] = P<int32_t>(c->col[m]);
        o->shift[m] = P<int8_t>(c->shift[m]);
    }
    return CRK_OK;
}

int64_t crk_launch_count(crk_ctx* c) { return c ? c->launches : -1; }

const char* crk_status_string(crk_status s) {
    switch (s) {
    case CRK_OK: return "ok";
    case CRK_EINVAL: return "invalid argument";
    case CRK_ENOMEM: return "out of device memory";
    case CRK_ECUDA: return "CUDA error";
    case CRK_ESTATE: return "call order violated";
    case CRK_ECAPACITY: return "capacity exceeded";
    }
    return "unknown status";
}

const char* crk_last_error(crk_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

}  // extern "C"
