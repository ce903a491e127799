// Frame workspace layout + the ordered (decoupled look-back) compaction scan.
#pragma once
#include "common.cuh"
#include "util.cuh"

namespace cinr {

constexpr int kTile = 256;        // rays per look-back tile (one per thread)
constexpr int kItersPerSm = 6;    // persistent CTAs per SM for an iteration kernel
constexpr int kMaxIterCap = 16383;

// Structure-of-arrays live-ray state, double buffered across iterations.
struct LiveBuf {
    int32_t* id;      // ray index into ray_* arrays, -1 = terminated
    long long* cur;   // cursor_f (as bits) when adaptive, else cursor_k
    double* col;      // [3n]
    double* tr;
};

struct FrameCounters {
    int ticket_rays;
    int nonfinite;
    int pad[14];
};

struct FrameWs {
    uint8_t* pix_keep;
    int32_t* ray_pix;
    double* ray_dir;
    double* ray_ten;
    double* ray_tex;
    LiveBuf buf[2];
    uint32_t* rng;
    int32_t* mq_slot;
    double* mq_pos;
    double* mq_dt;
    unsigned long long* status;
    int64_t max_tiles;
    int* live;      // [max_it+2] entries in the input buffer of iteration k
    int* ticket;    // [max_it+2] tile tickets per iteration
    int* nmiss;     // [max_it+2] true misses queued per iteration
    FrameCounters* ctr;
    void* ctr_iter;
    size_t ctr_iter_bytes;
};

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Carves the workspace (or only sizes it when base == nullptr).
inline int64_t frame_ws_layout(int64_t n, int32_t max_it, void* base, FrameWs* w) {
    if (max_it > kMaxIterCap) max_it = kMaxIterCap;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    const int64_t tiles = (n + kTile - 1) / kTile + 1 + 8 * 148 * 8;  // + G for even-tile rounding
    size_t o_keep = take((size_t)n);
    size_t o_pix = take((size_t)n * 4);
    size_t o_dir = take((size_t)n * 24);
    size_t o_ten = take((size_t)n * 8);
    size_t o_tex = take((size_t)n * 8);
    size_t o_b[2][4];
    for (int b = 0; b < 2; b++) {
        o_b[b][0] = take((size_t)n * 4);
        o_b[b][1] = take((size_t)n * 8);
        o_b[b][2] = take((size_t)n * 24);
        o_b[b][3] = take((size_t)n * 8);
    }
    size_t o_rng = take((size_t)n * 4);
    size_t o_mqs = take((size_t)n * 4);
    size_t o_mqp = take((size_t)n * 48);  // miss positions (v1) / advance outputs by slot (two-phase)
    size_t o_mqd = take((size_t)n * 8);
    size_t o_st = take((size_t)tiles * 16);  // look-back words (wave march: agg + incl)
    size_t o_ctr = take(sizeof(FrameCounters));
    size_t iter_bytes = (size_t)(max_it + 2) * 4 * 3;
    size_t o_it = take(iter_bytes);
    if (base && w) {
        char* p = (char*)base;
        w->pix_keep = (uint8_t*)(p + o_keep);
        w->ray_pix = (int32_t*)(p + o_pix);
        w->ray_dir = (double*)(p + o_dir);
        w->ray_ten = (double*)(p + o_ten);
        w->ray_tex = (double*)(p + o_tex);
        for (int b = 0; b < 2; b++) {
            w->buf[b].id = (int32_t*)(p + o_b[b][0]);
            w->buf[b].cur = (long long*)(p + o_b[b][1]);
            w->buf[b].col = (double*)(p + o_b[b][2]);
            w->buf[b].tr = (double*)(p + o_b[b][3]);
        }
        w->rng = (uint32_t*)(p + o_rng);
        w->mq_slot = (int32_t*)(p + o_mqs);
        w->mq_pos = (double*)(p + o_mqp);
        w->mq_dt = (double*)(p + o_mqd);
        w->status = (unsigned long long*)(p + o_st);
        w->max_tiles = tiles;
        w->ctr = (FrameCounters*)(p + o_ctr);
        w->ctr_iter = p + o_it;
        w->ctr_iter_bytes = iter_bytes;
        w->live = (int*)(p + o_it);
        w->ticket = w->live + (max_it + 2);
        w->nmiss = w->ticket + (max_it + 2);
    }
    return (int64_t)align_up(off, 256);
}

struct ScanSmem {
    long long tile;
    int warp_tot[kTile / 32];
    long long prefix;
};

constexpr unsigned long long kFlagA = 1ull << 30;
constexpr unsigned long long kFlagP = 2ull << 30;
constexpr unsigned long long kValMask = (1ull << 30) - 1;

// Block-wide exclusive scan of 0/1 flags for `tile`, extended across tiles in
// ticket order by a warp-parallel decoupled look-back on `status` (words tagged
// with `tag` so stale words from other iterations/frames are never consumed).
// Returns the inclusive total through this tile; `excl` = global rank.
__device__ __forceinline__ uint32_t ordered_scan(int flag, long long tile, unsigned long long* status, uint32_t tag,
                                                 ScanSmem& sm, long long& excl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) sm.warp_tot[warp] = __popc(bal);
    __syncthreads();
    int wbase = 0, btot = 0;
#pragma unroll
    for (int i = 0; i < kTile / 32; i++) {
        int t = sm.warp_tot[i];
        wbase += (i < warp) ? t : 0;
        btot += t;
    }
    const unsigned long long tagw = (unsigned long long)tag << 32;
    if (warp == 0) {
        if (tile == 0) {
            if (lane == 0) {
                st_volatile_u64(status, tagw | kFlagP | (unsigned long long)btot);
                sm.prefix = 0;
            }
        } else {
            if (lane == 0) st_volatile_u64(status + tile, tagw | kFlagA | (unsigned long long)btot);
            long long acc = 0;
            long long base = tile - 1;
            for (;;) {
                const long long idx = base - lane;
                unsigned long long s;
                if (idx >= 0) {
                    do {
                        s = ld_volatile_u64(status + idx);
                    } while ((s >> 32) != tag || (s & (3ull << 30)) == 0);
                } else {
                    s = kFlagP;  // virtual prefix 0 before tile 0
                }
                const bool isP = (s & (3ull << 30)) == kFlagP;
                const unsigned pm = __ballot_sync(0xffffffffu, isP);
                long long v = (long long)(s & kValMask);
                if (pm) {
                    const int first = __ffs(pm) - 1;
                    if (lane > first) v = 0;
                    acc += warp_sum(v);
                    break;
                }
                acc += warp_sum(v);
                base -= 32;
            }
            if (lane == 0) {
                st_volatile_u64(status + tile, tagw | kFlagP | (unsigned long long)(acc + btot));
                sm.prefix = acc;
            }
        }
    }
    __syncthreads();
    excl = sm.prefix + wbase + wpre;
    return (uint32_t)(sm.prefix + btot);
}

}  // namespace cinr
