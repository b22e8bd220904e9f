// work.cuh -- jagged work decomposition shared by the persistent tiled kernels.
//
// Work unit n = (user u, head h, query group g): the unit's history is split into
// T_u = ceil(L_u / 128) tiles.  Units are laid out user-major in a flat tile space
//   unit (u, hg) owns flat tiles [HG*uts[u] + hg*T_u, HG*uts[u] + (hg+1)*T_u),  HG = H * G,
// where uts[u] = sum_{u' < u} T_u' (computed on the device by launch_user_tiles).
// CTA c of a grid of C owns flat tiles [c*T/C, (c+1)*T/C) (stream-K style): every CTA gets the
// same number of tiles (+-1) whatever the length mix, and at most its first and last items are
// partial units.  Partial results go to workspace slots 2c (first item) and 2c+1 (last item);
// slot_unit[] records which unit each slot holds (-1 = unused) so the merge kernel can combine
// the run of slots of each split unit in ascending CTA order (deterministic).
#pragma once
#include <cstdint>

#include "internal.h"

namespace vista {

struct Item {
    int u;        // user
    int hg;       // h * G + g
    int t0, t1;   // tile range [t0, t1) within the unit
    int Tu;       // tiles of the unit
    bool first, last;
};

struct ItemIter {
    // Tile counts fit in 32 bits: sum L < 2^31 (TMA coordinates), so HG * sum T < 2^30.
    const int64_t* uts;
    int B, HG;
    int t, end;
    bool started;

    __device__ void init(const int64_t* uts_, int B_, int HG_, int cta, int num_ctas) {
        uts = uts_;
        B = B_;
        HG = HG_;
        const int T = HG * (int)uts[B];
        t = (int)(((unsigned long long)cta * (unsigned)T) / (unsigned)num_ctas);
        end = (int)(((unsigned long long)(cta + 1) * (unsigned)T) / (unsigned)num_ctas);
        started = false;
    }
    __device__ bool next(Item& it) {
        if (t >= end) return false;
        int lo = 0, hi = B - 1;
        while (lo < hi) {  // largest u with HG*uts[u] <= t
            const int mid = (lo + hi + 1) >> 1;
            if (HG * (int)uts[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const int base = HG * (int)uts[lo];
        const int Tu = (int)(uts[lo + 1] - uts[lo]);
        const unsigned r = (unsigned)(t - base);
        it.u = lo;
        it.hg = (int)(r / (unsigned)Tu);
        it.t0 = (int)(r - (unsigned)it.hg * (unsigned)Tu);
        const int n = min(end - t, Tu - it.t0);
        it.t1 = it.t0 + n;
        it.Tu = Tu;
        it.first = !started;
        started = true;
        t += n;
        it.last = (t >= end);
        return true;
    }
};

__device__ __forceinline__ bool item_complete(const Item& it) { return it.t0 == 0 && it.t1 == it.Tu; }

// First flat tile of CTA c's range, and the CTA whose range holds flat tile x (ranges as in ItemIter).
__device__ __forceinline__ int range_begin(int c, int T, int C) {
    return (int)(((unsigned long long)c * (unsigned)T) / (unsigned)C);
}
__device__ __forceinline__ int cta_of_tile(int x, int T, int C) {
    int c = (int)(((unsigned long long)x * (unsigned)C) / (unsigned)T);
    while (c + 1 < C && range_begin(c + 1, T, C) <= x) ++c;
    while (c > 0 && range_begin(c, T, C) > x) --c;
    return c;
}
// Workspace slot in which CTA c holds its partial of the unit whose flat tiles start at u0.
__device__ __forceinline__ int slot_of(int c, int c_lo, int u0, int T, int C) {
    return (c > c_lo || range_begin(c, T, C) >= u0) ? 2 * c : 2 * c + 1;
}
__device__ __forceinline__ int item_slot(const Item& it, int cta) { return it.first ? 2 * cta : 2 * cta + 1; }

}  // namespace vista
