// x-run merging shared by the 2-D x-run kernels (ACCUM, EDM, 2-D Life).
#pragma once

#include "smx_common.cuh"

namespace smx {

// One warp maps the KX consecutive blocks x0 .. x0+KX-1 of grid row wy
// lane-parallel (detail::sweep's map + Void filter + strict y-1,
// simulator.hpp:190-202) and merges the tiles that are x-adjacent in the data
// into runs: s_run[r] = {lowest tile x, tile y, length in tiles}. Chains go in
// either direction (RB's reflected half maps consecutive blocks to descending
// x): a lane continues the run when its x step (+1 or -1) repeats the previous
// lane's step, or the previous lane had none (it is the run's first tile).
// Every useful tile lands in exactly one run. Call with all 32 lanes.
template <int KIND, int KX>
__device__ __forceinline__ void strip_runs(const Geom& g, int x0, int wy, int (*s_run)[3], int* s_nruns) {
    static_assert(KX <= 32, "one warp maps the strip");
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int wx = x0 + lane;
    int valid = lane < KX && wx < g.ex;
    outcome<int> o{1, 0, 0, 0, 1, 0};
    if (valid) {
        o = map_block<KIND>(g, wx, wy, 0);
        valid = !o.is_void && (g.ty1 == 0 || (o.y >= g.ty0 && o.y < g.ty1));
    }
    const int px = __shfl_up_sync(FULL, o.x, 1);
    const int py = __shfl_up_sync(FULL, o.y, 1);
    const int pv = __shfl_up_sync(FULL, valid, 1);
    const int dx = o.x - px;
    const int step = (lane > 0 && valid && pv && py == o.y && (dx == 1 || dx == -1)) ? dx : 0;
    const int pstep = __shfl_up_sync(FULL, step, 1);
    const bool head = valid && !(step != 0 && (lane == 0 || pstep == 0 || pstep == step));
    const unsigned heads = __ballot_sync(FULL, head);
    const unsigned vmask = __ballot_sync(FULL, valid);
    const int nstep = __shfl_down_sync(FULL, step, 1);  // direction of the run from a head
    if (head) {
        const int r = __popc(heads & ((1u << lane) - 1u));
        const unsigned above = lane == 31 ? 0u : ~((2u << lane) - 1u);
        const unsigned stop = (heads | ~vmask) & above;
        const int end = stop ? __ffs(stop) - 1 : 32;
        const int len = end - lane;
        s_run[r][0] = (len > 1 && lane < 31 && nstep < 0) ? o.x - (len - 1) : o.x;
        s_run[r][1] = o.y;
        s_run[r][2] = len;
    }
    if (lane == 0) *s_nruns = __popc(heads);
}

// KS strips of KX blocks (x0 = (xs * KS + k) * KX, k < KS) of grid row wy,
// mapped concurrently by warps 0 .. KS-1, their run tables compacted into
// s_run[0 .. *s_total). Every thread of the CTA must call it (it ends with a
// __syncthreads). s_run holds KS * KX entries.
template <int KIND, int KX, int KS>
__device__ __forceinline__ void strips_runs(const Geom& g, int xs, int wy, int (*s_run)[3], int* s_nrun,
                                            int* s_total) {
    static_assert(KX <= 32, "one warp maps a strip");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp < KS) strip_runs<KIND, KX>(g, (xs * KS + warp) * KX, wy, s_run + warp * KX, &s_nrun[warp]);
    __syncthreads();
    if (warp == 0) {
        int off = s_nrun[0];
        for (int k = 1; k < KS; ++k) {
            const int n = s_nrun[k];  // <= KX <= 32: one lane per run, uniform syncs
            int a = 0, b = 0, c = 0;
            if (lane < n) a = s_run[k * KX + lane][0], b = s_run[k * KX + lane][1], c = s_run[k * KX + lane][2];
            __syncwarp();
            if (lane < n) s_run[off + lane][0] = a, s_run[off + lane][1] = b, s_run[off + lane][2] = c;
            __syncwarp();
            off += n;
        }
        if (lane == 0) *s_total = off;
    }
    __syncthreads();
}

// Row r of a strip's runs (rho rows per run) -> the with-diagonal cell row cy
// and its cell span [xlo, xhi) clipped to x <= y; false when empty.
__device__ __forceinline__ bool run_row(const int (*s_run)[3], int rr, int rho, int S, int* cy, int* xlo,
                                        int* xhi) {
    const int r = rr / rho, ly = rr - r * rho;
    *cy = s_run[r][1] * rho + ly;
    *xlo = s_run[r][0] * rho;
    *xhi = min((s_run[r][0] + s_run[r][2]) * rho, *cy + 1);
    return *cy <= S - 1 && *xlo < *xhi;
}

}  // namespace smx
