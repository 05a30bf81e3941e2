// ctx.h — private state of a crk_ctx (libcrksr.so).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/crksr.h"

namespace crk {

// Compile-time shape of the list-driven pair kernels.
constexpr int JMAX = 8;          // j-leaf size (gravity and gas): one staging slot group
constexpr int GRAV_NW = 8;       // warps per gravity CTA  (i-leaf <= GRAV_NW * GRAV_G)
constexpr int GRAV_G = 16;       // i-particles per warp (2 j-slots per warp step)
constexpr int HYD_NW = 8;        // warps per hydro CTA    (gas i-leaf <= HYD_NW * HYD_G)
constexpr int HYD_G = 8;         // gas i-particles per warp (4 j-slots per warp step)

// Growable device buffer (stream-ordered allocations).
struct Buf {
    void* p = nullptr;
    size_t cap = 0;
};

enum Stage : int { ST_NONE = 0, ST_LISTS = 1, ST_GEO = 2, ST_COR = 3, ST_EXT = 4 };

struct Layout {
    double q;        // position quantum L_max 2^-23
    float inv_q;     // 2^23 / L_max (exact)
    int cs;          // log2(cell_side / q)
    int cbits;       // bits per axis of a cell index
    int fbits;       // bits per axis of the in-cell Morton key
    int ncell[3];
    int64_t ncm;     // size of the dense Morton-indexed cell arrays = 2^(3 cbits)
    float L[3];      // box as fp32 (exact: powers of two)
    int dlo[3], dhi[3];  // owned cells [dlo, dhi)
    bool partial;        // domain smaller than the box (ghosts present)
};

}  // namespace crk

struct crk_ctx {
    crk_params prm;
    int device = 0;
    crk::Layout lay;
    int stage = crk::ST_NONE;
    int64_t n = 0, n_gas = 0;
    int64_t nleaf[4] = {0, 0, 0, 0};
    int64_t nent[2] = {0, 0};     // list capacity (entries allocated: the rows' upper bounds)
    int64_t nlist[2] = {0, 0};    // entries in the lists (set by csr_views)
    int64_t launches = 0;
    std::string err;

    // sort
    crk::Buf keys_a, keys_b, idx_a, idx_b, cub_tmp;
    // permute scratch (reused for all fields)
    crk::Buf scratch;
    // sorted-order packed (x, y, z, m)
    crk::Buf xm;
    // cells (dense, Morton-indexed)
    crk::Buf cell_start, cell_end;
    crk::Buf leaf_cnt;           // 4 * (ncm + 1) int32 counts -> offsets
    // gas ranks
    crk::Buf gflag, grank, gas_idx;
    // leaves (4 sets)
    crk::Buf lfirst[4], lcount[4], lbbox[4], lmaxh2[4], lcell[4];
    crk::Buf lbox8[4];           // padded boxes: (lo xyz, max H^2), (hi xyz, 0) per leaf
    crk::Buf dev_scalars;        // [0] float max H^2 ; [1..] int64 totals
    // lists (0 gravity, 1 hydro)
    crk::Buf rowlen[2], rowoff[2], col[2], shift[2];
    crk::Buf rowend[2];          // row a holds entries [rowoff[a], rowend[a]) (rows written at their bound)
    crk::Buf csroff[2];          // crk_list_view: compacted CSR row offsets
    crk::Buf erec[2];            // packed entries: int2 (first | (count-1) << 29, leaf | shift << 26)
    crk::Buf rclass;             // per gas i-leaf row: 1 = its hydro list holds a ghost j-leaf (crk_select_rows)
    crk::Buf gmask;              // gravity entries: uint8 mask of the i-groups (16 i) of the row's leaf the entry
                                 // can reach (box test + Newton-3 / ghost rule), + 256 B pad for word reads
    // gas-ordered state
    crk::Buf gpos;               // float4 (x, y, z, H)
    crk::Buf gvel;               // float4 (vx, vy, vz, m)
    crk::Buf gV;                 // float
    crk::Buf gposV;              // float4 (x, y, z, V) j-rows of corrections/extras
    crk::Buf gcoef;              // 16 planes: A, B(3), dA(3), dB(9)  (A, dA unscaled)
    crk::Buf grec;               // accel records: 9 float4 per gas particle
    crk::Buf gu;                 // float
    crk::Buf gacc;               // float4 force accumulator (symmetric kernels)
    crk::Buf pinned;             // host pinned totals (mapped: written by k_readback, no copy engine)
    void* pinned_dev = nullptr;  // device alias of `pinned`
    crk::Buf sel_flag, sel_mask; // selection scratch
    crk::Buf work;               // dynamic work counters of the persistent kernels
    // gas neighbour lists (geometry -> corrections, extras, accel): pairs.cuh ListView
    crk::Buf nbr, ncnt, lflag;
    int nbr_cap = 0;             // entries per gas particle (0: lists off)
    // skin lists (crk_params.skin > 0): valid lists survive drifts until crk_refresh
    bool skin_lists = false;     // the last build used the skin and no rebuild is due
    bool csr_views = false;      // col / shift decoded for crk_list_view since the last build
    int row_sel = 0;             // crk_select_rows: 0 all rows, 1 interior rows, 2 rows holding ghosts
    crk::Buf disp;               // device floats: [0] this drift's max |dt v|, [1] bound since the build
};
