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
    int row0;     // offsets[u] (history row of the unit's first item; < 2^31)
    int len;      // L_u
    bool first, last;
};

// Largest u with HG * uts[u] <= t (t < HG * uts[B]); binary search, used once per walk.
__device__ __forceinline__ int user_of_tile(const int64_t* uts, int B, int HG, int t) {
    int lo = 0, hi = B - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (HG * (int)uts[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// The same search by a whole warp (all 32 lanes, converged): 32 probes per round, so B <= 1024
// users take two dependent loads instead of log2(B) -- the first item of a persistent CTA is on its
// start-up path.  Requires uts non-decreasing and uts[0] = 0.
__device__ __forceinline__ int user_of_tile_w(const int64_t* uts, int B, int HG, int t) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = B - 1;  // invariant: HG * uts[lo] <= t; the answer is in [lo, hi]
    while (hi - lo >= 32) {
        const int step = (hi - lo + 32) / 32;
        const int pos = min(lo + lane * step, hi);
        const unsigned m = __ballot_sync(0xffffffffu, HG * (int)uts[pos] <= t);
        const int k = 31 - __clz(m);  // last probe that holds (lane 0 always does)
        const int nlo = min(lo + k * step, hi);
        hi = k < 31 ? min(lo + (k + 1) * step - 1, hi) : hi;
        lo = nlo;
    }
    const int pos = lo + lane;
    const unsigned m = __ballot_sync(0xffffffffu, pos <= hi && HG * (int)uts[min(pos, hi)] <= t);
    return lo + 31 - __clz(m);
}

struct ItemIter {
    // Tile counts fit in 32 bits: sum L < 2^31 (TMA coordinates), so HG * sum T < 2^30.
    // One binary search at the first item; afterwards the walk advances user by user (a CTA's
    // range is contiguous), one uts[] load per user boundary instead of a log2(B)-deep search.
    // uts / B / HG come from the kernel parameters at every call (no registers held for them).
    int t, end;
    int u, base, Tu;  // current user (-1 before the first item), its first flat tile, tiles per unit
    bool wsearch;     // every call is made by a full, converged warp: warp-wide first search

    __device__ void init(const int64_t* uts, int B, int HG, int cta, int num_ctas, bool warp_wide = false) {
        const int T = HG * (int)uts[B];
        t = (int)(((unsigned long long)cta * (unsigned)T) / (unsigned)num_ctas);
        end = (int)(((unsigned long long)(cta + 1) * (unsigned)T) / (unsigned)num_ctas);
        u = -1;
        wsearch = warp_wide;
    }
    __device__ bool next(Item& it, const int64_t* uts, int B, int HG) {
        if (t >= end) return false;
        it.first = u < 0;
        if (u < 0) {
            u = wsearch ? user_of_tile_w(uts, B, HG, t) : user_of_tile(uts, B, HG, t);
            const int a = (int)uts[u];
            base = HG * a;
            Tu = (int)uts[u + 1] - a;
        }
        while (t >= base + HG * Tu) {  // next non-empty user (t < end <= HG * uts[B] bounds this)
            ++u;
            base += HG * Tu;
            Tu = (int)uts[u + 1] - base / HG;
        }
        const unsigned r = (unsigned)(t - base);
        it.u = u;
        it.hg = (int)(r / (unsigned)Tu);
        it.t0 = (int)(r - (unsigned)it.hg * (unsigned)Tu);
        const int n = min(end - t, Tu - it.t0);
        it.t1 = it.t0 + n;
        it.Tu = Tu;
        t += n;
        it.last = (t >= end);
        return true;
    }
};

// Units held in CTA c's partial slots 2c (first item) / 2c+1 (last item), -1 if that item is a
// whole unit or absent.  Only the first and the last item of a range can be partial, so this
// looks at those two directly instead of walking the range.
__device__ __forceinline__ void partial_slots(const int64_t* uts, int B, int HG, int cta, int num_ctas, int& s0,
                                              int& s1) {
    s0 = s1 = -1;
    const int T = HG * (int)uts[B];
    const int beg = (int)(((unsigned long long)cta * (unsigned)T) / (unsigned)num_ctas);
    const int end = (int)(((unsigned long long)(cta + 1) * (unsigned)T) / (unsigned)num_ctas);
    if (beg >= end) return;
    // first item: unit holding tile beg
    int u = user_of_tile(uts, B, HG, beg);
    int a = (int)uts[u], Tu = (int)uts[u + 1] - a;
    int r = beg - HG * a, hg = r / Tu;
    const int f_start = HG * a + hg * Tu, f_end = f_start + Tu;
    if (beg > f_start || end < f_end) s0 = u * HG + hg;
    if (end <= f_end) return;  // one item only
    // last item: unit holding tile end-1 (starts inside the range, so partial iff cut at end)
    u = user_of_tile(uts, B, HG, end - 1);
    a = (int)uts[u];
    Tu = (int)uts[u + 1] - a;
    r = end - 1 - HG * a;
    hg = r / Tu;
    if (end < HG * a + (hg + 1) * Tu) s1 = u * HG + hg;
}

#ifndef VISTA_GMAJOR
#define VISTA_GMAJOR 1
#endif
// Query-group-major work order for a kernel whose units re-read a user's K/V once per query group
// (the softmax backward dQ pass, G = S / 128); 0 = unit-major.  Measured on the forward at S = 512
// too: +1% at c5, but the generic iterator cost 2% at c2 (G = 1), so the forward keeps ItemIter.
constexpr int kGMajor = VISTA_GMAJOR;
__device__ __forceinline__ int gmajor_groups(int G, int num_ctas) { return (kGMajor && G > 1 && num_ctas % G == 0) ? G : 1; }

struct ItemIterG {
    // ItemIter with an optional query-group-major order.
    // G > 1 (query-group-major order, "g-major"): the flat space is G blocks of H * uts[B] tiles,
    // block g holding the units (u, h, g) user-major.  With C divisible by G, CTAs c and
    // c + C/G, ... walk the same (user, head, tile) sequence for the G query groups at the same
    // time, so each K/V tile is fetched from HBM once and hit in L2 by the other groups.
    int t, end;
    int u, base, Tu;  // current user (-1 before the first item), its first flat tile, tiles per unit
    int G, g;         // query groups per head (1: unit-major order), current group

    __device__ void init(const int64_t* uts, int B, int HG, int cta, int num_ctas, int groups = 1) {
        const int T = HG * (int)uts[B];
        t = (int)(((unsigned long long)cta * (unsigned)T) / (unsigned)num_ctas);
        end = (int)(((unsigned long long)(cta + 1) * (unsigned)T) / (unsigned)num_ctas);
        u = -1;
        G = groups;
        g = 0;
    }
    __device__ bool next(Item& it, const int64_t* uts, int B, int HG) {
        if (t >= end) return false;
        const int H = G > 1 ? HG / G : HG;
        it.first = u < 0;
        if (u < 0) {
            int tl = t;
            if (G > 1) {
                const int TH = H * (int)uts[B];
                g = t / TH;
                tl = t - g * TH;
            }
            u = user_of_tile(uts, B, H, tl);
            const int a = (int)uts[u];
            base = (t - tl) + H * a;
            Tu = (int)uts[u + 1] - a;
        }
        while (t >= base + H * Tu) {  // next non-empty user (t < end <= HG * uts[B] bounds this)
            base += H * Tu;
            if (++u == B) {  // g-major: wrap to the next query group's block
                u = 0;
                ++g;
            }
            Tu = (int)(uts[u + 1] - uts[u]);
        }
        const unsigned r = (unsigned)(t - base);
        const int h = (int)(r / (unsigned)Tu);
        it.u = u;
        it.hg = G > 1 ? h * G + g : h;
        it.t0 = (int)(r - (unsigned)h * (unsigned)Tu);
        const int n = min(end - t, Tu - it.t0);
        it.t1 = it.t0 + n;
        it.Tu = Tu;
        t += n;
        it.last = (t >= end);
        return true;
    }
};

// Units held in CTA c's partial slots 2c (first item) / 2c+1 (last item), -1 if that item is a
// whole unit or absent.  Only the first and the last item of a range can be partial, so this
// looks at those two directly instead of walking the range.  G as in ItemIterG.
__device__ __forceinline__ void unit_at(const int64_t* uts, int B, int HG, int G, int x, int& n, int& f_start,
                                        int& f_end) {
    const int H = G > 1 ? HG / G : HG;
    int g = 0, tl = x;
    if (G > 1) {
        const int TH = H * (int)uts[B];
        g = x / TH;
        tl = x - g * TH;
    }
    const int u = user_of_tile(uts, B, H, tl);
    const int a = (int)uts[u], Tu = (int)uts[u + 1] - a;
    const int h = (tl - H * a) / Tu;
    f_start = (x - tl) + H * a + h * Tu;
    f_end = f_start + Tu;
    n = u * HG + (G > 1 ? h * G + g : h);
}
__device__ __forceinline__ void partial_slots_g(const int64_t* uts, int B, int HG, int cta, int num_ctas, int& s0,
                                              int& s1, int G) {
    s0 = s1 = -1;
    const int T = HG * (int)uts[B];
    const int beg = (int)(((unsigned long long)cta * (unsigned)T) / (unsigned)num_ctas);
    const int end = (int)(((unsigned long long)(cta + 1) * (unsigned)T) / (unsigned)num_ctas);
    if (beg >= end) return;
    int n, f_start, f_end;
    unit_at(uts, B, HG, G, beg, n, f_start, f_end);  // first item: the unit holding tile beg
    if (beg > f_start || end < f_end) s0 = n;
    if (end <= f_end) return;  // one item only
    unit_at(uts, B, HG, G, end - 1, n, f_start, f_end);  // last item: starts inside the range
    if (end < f_end) s1 = n;
}

__device__ __forceinline__ bool item_complete(const Item& it) { return it.t0 == 0 && it.t1 == it.Tu; }

__device__ __forceinline__ int item_slot(const Item& it, int cta) { return it.first ? 2 * cta : 2 * cta + 1; }

}  // namespace vista
