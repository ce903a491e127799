// Between-frame maintenance on device (session.py:132-142), bit-exact with the
// reference's single-writer Python logic:
//   k_report      Mrpd.drain_miss_reports + RequestTable.report_many
//                 (mrpd.py:263-266, scheduler.py:60-72): new key -> base=f,
//                 hits=c-1; existing -> hits+=c (order-independent)
//   k_insert      InlineLoader.collect + Mrpd.insert (mrpd.py:229-256) with
//                 BrickPool.acquire_slot (pool.py:55-62): free slots ascending,
//                 then argmin(last_used) over last_used < f, lowest slot on ties,
//                 else deferred; the LRU picks of one batch are the m smallest
//                 (last_used, slot) keys, found by a block radix select
//   k_pending +   RequestTable.select_batch (scheduler.py:79-101): composite
//   k_select      64-bit key (-rank|base, linear, lod); the smallest prefix holding
//                 n non-excluded (mapped) entries is deleted, its non-excluded
//                 entries returned in key order
//   field decode  fulfill (scheduler.py:127-134) into the staging slab; a
//                 non-finite decode re-enters the keys with base=f (164-168)
#include <cstddef>
#include <vector>

#include "common.cuh"
#include "fields.cuh"
#include "util.cuh"

namespace cinr {

constexpr int kSelThreads = 1024;
constexpr int kMaxSel = 2048;  // max_requests bound for the in-CTA selection

struct MaintWs {
    long long* pend_key;   // [total]
    long long* pend_flat;  // [total]
    int* ctr;              // [0] n_pending, [1] n_reports
    long long* lru;        // [kMaxSel]
    int* assign;           // [kMaxSel]
    int* nonfinite;        // [0] decode flag, [1] skip (the frame failed), [2..3] bricks to decode (i64)
    __host__ __device__ long long* n_dec() const { return reinterpret_cast<long long*>(nonfinite + 2); }
};

// The frame just rendered raised a non-finite inference: the reference raises
// RenderError before _maintenance (sampler.py:149-152), so nothing here may run.
__device__ __forceinline__ bool maint_skipped(const MaintWs& w) { return w.nonfinite[1] != 0; }

inline int64_t maint_ws_layout(int64_t total, void* base, MaintWs* w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = (off + 255) / 256 * 256;
        off = o + bytes;
        return o;
    };
    size_t a = take((size_t)total * 8), b = take((size_t)total * 8), c = take(64), d = take(kMaxSel * 8),
           e = take(kMaxSel * 4), f = take(64);
    if (base && w) {
        char* p = (char*)base;
        w->pend_key = (long long*)(p + a);
        w->pend_flat = (long long*)(p + b);
        w->ctr = (int*)(p + c);
        w->lru = (long long*)(p + d);
        w->assign = (int*)(p + e);
        w->nonfinite = (int*)(p + f);
    }
    return (int64_t)((off + 255) / 256 * 256);
}

__device__ __forceinline__ int lod_of(const VcbBrickGeom& G, long long flat) {
    int lod = 0;
    while (lod + 1 < G.n_lod && flat >= G.offset[lod + 1]) lod++;
    return lod;
}

__global__ void k_maint_gate(VcbMaintParams P, MaintWs w) {
#pragma unroll
    for (int i = 0; i < 16; i++) w.ctr[i] = 0;  // [0] n_pending, [1] n_reports (64 B)
    w.nonfinite[0] = 0;
    w.nonfinite[1] = (P.frame_stats != nullptr && P.frame_stats->nonfinite != 0) ? 1 : 0;
    *w.n_dec() = 0;
}

// drain_miss_reports + report_many (mrpd.py:263, scheduler.py:60-72): a scan of the
// per-brick counters, four at a time (the frame kernels' fire-and-forget reductions
// stay cheap that way; 78 MB at 4096^3@B16); a key new to the request table joins the
// pending list
__device__ __forceinline__ void report_brick(const VcbMaintParams& P, long long b, int c) {
    P.miss_count[b] = 0;
    if (P.req_base[b] < 0) {
        P.req_base[b] = P.session_frame;
        P.req_hits[b] = c - 1;
        if (P.list_counts != nullptr) P.pending_list[atomicAdd(P.list_counts + 1, 1)] = (int32_t)b;
    } else {
        P.req_hits[b] += c;
    }
}

__global__ void k_report(VcbMaintParams P, MaintWs w) {
    if (maint_skipped(w)) return;
    const long long n4 = P.total >> 2;
    const int4* mc4 = reinterpret_cast<const int4*>(P.miss_count);  // cudaMalloc'd: 16-byte aligned
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n4;
         i += (long long)gridDim.x * blockDim.x) {
        int c4[4];
        if (i < n4) {
            const int4 v = __ldcs(mc4 + i);
            c4[0] = v.x;
            c4[1] = v.y;
            c4[2] = v.z;
            c4[3] = v.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++) c4[q] = (4 * i + q < P.total) ? P.miss_count[4 * i + q] : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int c = c4[q];
            if (c == 0) continue;
            const long long b = 4 * i + q;
            report_brick(P, b, c);
            const int r = atomicAdd(&w.ctr[1], 1);
            if (P.dbg_reports) {
                P.dbg_reports[2 * r] = b;
                P.dbg_reports[2 * r + 1] = c;
            }
        }
    }
}

// Smallest-m selection of unique 64-bit keys by one CTA: one pass finds the
// candidates' key range, then an MSB-first radix select with 11-bit digits over the
// key offsets (k - kmin: the spread, not the 64-bit width, sets the pass count --
// 2-3 passes for the LRU and request-table keys), the digit holding the m-th key
// found by a block scan of the histogram; the <= threshold keys are gathered and
// rank-sorted.
constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;  // = 2 * kSelThreads
static_assert(kBins == 2 * kSelThreads, "two histogram bins per thread");

struct SelSmem {
    unsigned int hist[kBins];
    unsigned int warp_sum[kSelThreads / 32];
    unsigned long long prefix, mask, kmin, kmax;
    long long remaining, ncand;
    int n_out;
    long long out[kMaxSel];
};

// exclusive block scan of one value per thread (blockDim = kSelThreads)
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* warp_sum) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned t = warp_sum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        warp_sum[lane] = t - warp_sum[lane];  // exclusive warp offsets
    }
    __syncthreads();
    return x - v + warp_sum[wid];
}

template <typename KeyFn>
__device__ int block_select_smallest(KeyFn key_of, long long n, int m, SelSmem& s, long long* sorted_out) {
    // key_of(i, &k) -> false when element i is not a candidate
    if (threadIdx.x == 0) {
        s.prefix = 0;
        s.mask = 0;
        s.remaining = m;
        s.n_out = 0;
        s.kmin = ~0ull;
        s.kmax = 0;
        s.ncand = 0;
    }
    __syncthreads();
    unsigned long long kmin = ~0ull, kmax = 0;
    long long nc = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        unsigned long long k;
        if (key_of(i, k)) {
            kmax = k > kmax ? k : kmax;
            kmin = k < kmin ? k : kmin;
            nc++;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmax, o), b = __shfl_xor_sync(0xffffffffu, kmin, o);
        kmax = a > kmax ? a : kmax;
        kmin = b < kmin ? b : kmin;
        nc += __shfl_xor_sync(0xffffffffu, nc, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&s.kmax, kmax);
        atomicMin(&s.kmin, kmin);
        atomicAdd((unsigned long long*)&s.ncand, (unsigned long long)nc);
    }
    __syncthreads();
    const long long ncand = s.ncand;
    const unsigned long long base = s.kmin;
    unsigned long long thresh = ~0ull;
    if (ncand > m) {
        const unsigned long long span = s.kmax - base;  // > 0: keys are unique, ncand >= 2
        const int bits = 64 - __clzll((long long)span);
        int shift = ((bits + kDigitBits - 1) / kDigitBits) * kDigitBits;
        while (shift > 0) {
            shift -= kDigitBits;
            s.hist[threadIdx.x] = 0;
            s.hist[threadIdx.x + kSelThreads] = 0;
            __syncthreads();
            const unsigned long long pf = s.prefix, mk = s.mask;
            const long long rem = s.remaining;
            for (long long i = threadIdx.x; i < n; i += blockDim.x) {
                unsigned long long k;
                if (key_of(i, k)) {
                    const unsigned long long r = k - base;
                    if ((r & mk) == pf) atomicAdd(&s.hist[(r >> shift) & (kBins - 1)], 1u);
                }
            }
            __syncthreads();
            const unsigned a = s.hist[2 * threadIdx.x], b = s.hist[2 * threadIdx.x + 1];
            const long long ex = block_excl_scan(a + b, s.warp_sum);
            // exactly one thread's pair of bins holds the rem-th key
            if (ex < rem && ex + a + b >= rem) {
                const bool first = ex + a >= rem;
                const unsigned long long d = 2ull * threadIdx.x + (first ? 0 : 1);
                s.remaining = first ? rem - ex : rem - ex - a;
                s.prefix = pf | (d << shift);
                s.mask = mk | ((unsigned long long)(kBins - 1) << shift);
            }
            __syncthreads();
        }
        thresh = base + s.prefix;  // the m-th smallest key
    }
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        unsigned long long k;
        if (key_of(i, k) && k <= thresh) {
            int o = atomicAdd(&s.n_out, 1);
            if (o < kMaxSel) s.out[o] = (long long)k;
        }
    }
    __syncthreads();
    const int cnt = s.n_out < kMaxSel ? s.n_out : kMaxSel;
    // rank sort (keys unique)
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const long long k = s.out[i];
        int r = 0;
        for (int j = 0; j < cnt; j++) r += s.out[j] < k;
        sorted_out[r] = k;
    }
    __syncthreads();
    return cnt;
}

__global__ void __launch_bounds__(kSelThreads) k_insert(VcbMaintParams P, MaintWs w) {
    __shared__ SelSmem s;
    __shared__ long long n_lru_s;
    if (maint_skipped(w)) return;
    VcbCacheState* st = P.state;
    const long long n = st->n_staged;
    if (n == 0) {
        if (threadIdx.x == 0) {
            st->bricks_loaded = 0;
            st->deferred = 0;
            st->inserted = 0;
        }
        return;
    }
    const long long f = P.session_frame;
    const long long nf0 = st->next_free;
    const long long free_left = P.slots - nf0;
    // entries already mapped are refreshed in place (mrpd.py:240-243); their slots are
    // stashed in w.assign (each thread revisits only its own entries below)
    __shared__ int n_exist_s;
    if (threadIdx.x == 0) n_exist_s = 0;
    __syncthreads();
    int ne = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const int e = P.table[P.staged_keys[i]];
        w.assign[i] = e;
        ne += e >= 0;
    }
    for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
    if ((threadIdx.x & 31) == 0 && ne) atomicAdd(&n_exist_s, ne);
    // LRU candidates only matter when the free list cannot cover the batch
    long long n_lru = 0;
    if (n > free_left) {
        int slot_bits = 1;
        while ((1ll << slot_bits) < P.slots) slot_bits++;
        auto key_of = [&](long long i, unsigned long long& k) -> bool {
            const long long lu = P.last_used[i];
            if (lu >= f) return false;
            k = ((unsigned long long)(lu + 1) << slot_bits) | (unsigned long long)i;
            return true;
        };
        const int m = (int)(n < kMaxSel ? n : kMaxSel);
        int cnt = block_select_smallest(key_of, nf0, m, s, w.lru);
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) w.lru[i] &= (1ll << slot_bits) - 1;
        n_lru = cnt;
    }
    if (threadIdx.x == 0) n_lru_s = n_lru;
    __syncthreads();
    if (n_exist_s == 0 || n <= free_left) {
        // no refreshed slot can be an LRU pick, so entries do not interact: the r-th new
        // key (batch order) takes the r-th free slot (pool.py:55-58), then the r-th
        // oldest (last_used, slot) (pool.py:59-62), else it is deferred
        __shared__ int chunk_new_s;
        long long new_before = 0;
        for (long long c0 = 0; c0 < n; c0 += blockDim.x) {
            const long long i = c0 + threadIdx.x;
            const int existing = i < n ? w.assign[i] : 0;
            const bool fresh = i < n && existing < 0;
            const unsigned rk = block_excl_scan(fresh ? 1u : 0u, s.warp_sum);
            if (threadIdx.x == blockDim.x - 1) chunk_new_s = (int)rk + (fresh ? 1 : 0);
            if (i < n) {
                int slot = existing;
                if (fresh) {
                    const long long r = new_before + rk;
                    const long long key = P.staged_keys[i];
                    slot = r < free_left ? (int)(nf0 + r) : (r - free_left < n_lru ? (int)w.lru[r - free_left] : -1);
                    if (slot >= 0) {
                        const long long old = P.owner[slot];
                        if (old >= 0) P.table[old] = -1;
                        P.owner[slot] = key;
                        P.table[key] = slot;
                    }
                }
                if (slot >= 0) P.last_used[slot] = f;
                w.assign[i] = slot;
            }
            __syncthreads();
            new_before += chunk_new_s;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const long long from_free = new_before < free_left ? new_before : free_left;
            const long long from_lru = new_before - from_free < n_lru ? new_before - from_free : n_lru;
            st->next_free = nf0 + from_free;
            st->bricks_loaded = (n - new_before) + from_free + from_lru;
            st->deferred = new_before - from_free - from_lru;
            st->inserted = from_free + from_lru;
            st->loaded_total += from_free + from_lru;
        }
    } else if (threadIdx.x == 0) {
        long long next_free = nf0, lp = 0, loaded = 0, deferred = 0, inserted = 0;
        for (long long i = 0; i < n; i++) {
            const long long key = P.staged_keys[i];
            const int existing = P.table[key];
            int slot = -1;
            if (existing >= 0) {
                slot = existing;
                P.last_used[slot] = f;
                w.assign[i] = slot;
                loaded++;
                continue;
            }
            if (next_free < P.slots) {
                slot = (int)next_free++;
            } else {
                while (lp < n_lru_s && P.last_used[w.lru[lp]] >= f) lp++;
                if (lp < n_lru_s) slot = (int)w.lru[lp++];
            }
            if (slot < 0) {
                deferred++;
                w.assign[i] = -1;
                continue;
            }
            const long long old = P.owner[slot];
            if (old >= 0) P.table[old] = -1;
            P.owner[slot] = key;
            P.table[key] = slot;
            P.last_used[slot] = f;
            w.assign[i] = slot;
            inserted++;
            loaded++;
        }
        st->next_free = next_free;
        st->bricks_loaded = loaded;
        st->deferred = deferred;
        st->inserted = inserted;
        st->loaded_total += inserted;
    }
    __syncthreads();
    const long long b3 = P.geom.b * P.geom.b * P.geom.b;
    for (long long i = 0; i < n; i++) {
        const int slot = w.assign[i];
        if (slot < 0) continue;
        const float4* src = reinterpret_cast<const float4*>(P.staging + i * b3);
        float4* dst = reinterpret_cast<float4*>(P.pool + (long long)slot * b3);
        if ((b3 & 3) == 0) {
            for (long long t = threadIdx.x; t < b3 / 4; t += blockDim.x) dst[t] = src[t];
        } else {
            for (long long t = threadIdx.x; t < b3; t += blockDim.x) P.pool[(long long)slot * b3 + t] = P.staging[i * b3 + t];
        }
    }
}

__device__ __forceinline__ unsigned long long composite_key(const VcbMaintParams& P, long long b) {
    const int lod = lod_of(P.geom, b);
    const unsigned long long lin = (unsigned long long)(b - P.geom.offset[lod]);
    const int low = P.lin_bits + P.lod_bits;
    const long long base = P.req_base[b];
    unsigned long long hi;
    if (P.ranking) {
        const long long h = P.req_hits[b];
        const long long r = (base + h < base + P.rank_clamp) ? base + h : base + P.rank_clamp;
        const unsigned long long rmax = (1ull << (63 - low)) - 1;
        hi = rmax - (unsigned long long)r;
    } else {
        hi = (unsigned long long)base;
    }
    return (hi << low) | (lin << P.lod_bits) | (unsigned long long)lod;
}

__global__ void k_pending(VcbMaintParams P, MaintWs w) {
    if (maint_skipped(w)) return;
    if (P.list_counts != nullptr) {
        // the pending list holds exactly the keys with req_base >= 0
        const long long n = P.list_counts[1];
        if (blockIdx.x == 0 && threadIdx.x == 0) w.ctr[0] = (int)n;
        for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n;
             o += (long long)gridDim.x * blockDim.x) {
            const long long b = P.pending_list[o];
            w.pend_flat[o] = b;
            w.pend_key[o] = (long long)composite_key(P, b) | (P.table[b] >= 0 ? (1ll << 63) : 0ll);
        }
        return;
    }
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < P.total;
         b += (long long)gridDim.x * blockDim.x) {
        if (P.req_base[b] < 0) continue;
        const int o = atomicAdd(&w.ctr[0], 1);
        w.pend_flat[o] = b;
        // excluded (is_mapped) entries carry the top bit so a selection over
        // non-excluded keys can skip them
        w.pend_key[o] = (long long)composite_key(P, b) | (P.table[b] >= 0 ? (1ll << 63) : 0ll);
    }
}

__global__ void __launch_bounds__(kSelThreads) k_select(VcbMaintParams P, MaintWs w) {
    __shared__ SelSmem s;
    __shared__ long long picked[kMaxSel];
    if (maint_skipped(w)) return;
    VcbCacheState* st = P.state;
    const long long np = w.ctr[0];
    int m = P.max_requests < kMaxSel ? P.max_requests : kMaxSel;
    if (P.decode_budget >= 0) {
        // frame scheduler: the frame's decoded true misses came first; the batch gets the
        // rest of the per-frame sample budget, at least one brick so the cache progresses
        const long long b3 = P.geom.b * P.geom.b * P.geom.b;
        const long long used = P.frame_stats != nullptr ? P.frame_stats->misses_resolved : 0;
        long long nb = (P.decode_budget - used) / b3;
        if (nb < 1) nb = 1;
        if (nb < m) m = (int)nb;
    }
    auto key_ok = [&](long long i, unsigned long long& k) -> bool {
        const long long v = w.pend_key[i];
        if (v < 0) return false;  // excluded (mapped)
        k = (unsigned long long)v;
        return true;
    };
    const int cnt = block_select_smallest(key_ok, np, m, s, picked);
    // threshold: the last picked key when n were found, else everything goes
    const unsigned long long thresh = (cnt >= m && cnt > 0) ? (unsigned long long)picked[cnt - 1] : ~0ull;
    for (long long i = threadIdx.x; i < np; i += blockDim.x) {
        const unsigned long long k = (unsigned long long)w.pend_key[i] & ~(1ull << 63);
        if (k <= thresh) P.req_base[w.pend_flat[i]] = -1;  // popped (returned or dropped)
    }
    if (P.list_counts != nullptr) {
        // the surviving entries form the next pending list (w.pend_flat holds this one)
        __shared__ int n_keep;
        if (threadIdx.x == 0) n_keep = 0;
        __syncthreads();
        for (long long i = threadIdx.x; i < np; i += blockDim.x) {
            const long long b = w.pend_flat[i];
            if (P.req_base[b] >= 0) P.pending_list[atomicAdd(&n_keep, 1)] = (int32_t)b;
        }
        __syncthreads();
        if (threadIdx.x == 0) P.list_counts[1] = n_keep;
    }
    const unsigned long long lowmask = (1ull << (P.lin_bits + P.lod_bits)) - 1;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const unsigned long long k = (unsigned long long)picked[i] & lowmask;
        const int lod = (int)(k & ((1ull << P.lod_bits) - 1));
        const long long lin = (long long)(k >> P.lod_bits);
        P.staged_keys[i] = P.geom.offset[lod] + lin;
    }
    if (threadIdx.x == 0) {
        *w.n_dec() = cnt;
        st->n_staged = cnt;
        st->staged_frame = P.session_frame;
        st->n_inflight = cnt;
        st->n_pending = np;
        st->n_batch = cnt;
        st->n_reports = w.ctr[1];
    }
}

int inr_bricks_tc_dev(const VcbField& F, const VcbBrickGeom& G, const int64_t* keys, const int64_t* n_keys_dev,
                      int max_keys, float* out, int32_t* nonfinite, cudaStream_t st);

template <int kInr>
__global__ void k_decode_bricks_dev(VcbField F, VcbBrickGeom G, const int64_t* keys, const int64_t* n_keys_dev,
                                    int max_keys, float* out, int* nonfinite) {
    extern __shared__ __align__(16) float smem[];
    MlpSmem m;
    const long long nk = *n_keys_dev;
    if (nk == 0) return;
    if (F.kind == 0) {
        stage_mlp(F, smem, m);
        __syncthreads();
    }
    const long long b = G.b, b3 = b * b * b;
    const long long total = nk * b3;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long ki = t / b3, s_ = t - ki * b3;
        const long long flat = keys[ki];
        const int lod = lod_of(G, flat);
        const long long lin = flat - G.offset[lod];
        const long long gx = G.grid[lod][0], gy = G.grid[lod][1];
        const long long ix = lin % gx, iy = (lin / gx) % gy, iz = lin / (gx * gy);
        const long long x = s_ % b, y = (s_ / b) % b, z = s_ / (b * b);
        long long nx = (ix > 0 ? ix * (b << lod) - 1 : 0) + (x << lod);
        long long ny = (iy > 0 ? iy * (b << lod) - 1 : 0) + (y << lod);
        long long nz = (iz > 0 ? iz * (b << lod) - 1 : 0) + (z << lod);
        nx = nx < G.dims[0] - 1 ? nx : G.dims[0] - 1;
        ny = ny < G.dims[1] - 1 ? ny : G.dims[1] - 1;
        nz = nz < G.dims[2] - 1 ? nz : G.dims[2] - 1;
        int bad = 0;
        out[t] = field_eval<kInr>(F, ((double)nx + 0.5) / (double)G.dims[0], ((double)ny + 0.5) / (double)G.dims[1],
                                   ((double)nz + 0.5) / (double)G.dims[2], m, &bad);
        if (bad) *nonfinite = 1;
    }
}

__global__ void k_post_decode(VcbMaintParams P, MaintWs w) {
    if (maint_skipped(w)) return;
    VcbCacheState* st = P.state;
    if (*w.nonfinite) {
        // InlineLoader.dispatch failure: keys re-enter with base = f, hits = 0
        for (long long i = 0; i < st->n_staged; i++) {
            const long long b = P.staged_keys[i];
            if (P.list_counts != nullptr && P.req_base[b] < 0)
                P.pending_list[P.list_counts[1]++] = (int32_t)b;
            P.req_base[b] = P.session_frame;
            P.req_hits[b] = 0;
        }
        st->n_staged = 0;
        st->n_inflight = 0;
        st->decode_error += 1;
        *w.nonfinite = 0;
    }
}

int mlp_smem_bytes(const VcbField& F);
extern thread_local long long g_launches;

}  // namespace cinr

using namespace cinr;

extern "C" int64_t vcb_maint_workspace_bytes(int64_t total_bricks, int64_t slots, int32_t max_requests) {
    (void)slots;
    (void)max_requests;
    return maint_ws_layout(total_bricks, nullptr, nullptr);
}

// fulfill (scheduler.py:127-134) of the batch k_select staged (w.n_dec keys, 0 when the
// maintenance was skipped) into the staging slab, then the failure path (k_post_decode)
// Decode bricks `keys` (count on the device) of P's field into `out` ([max_keys][B^3]).
static void decode_keys(const VcbMaintParams& P, const int64_t* keys, const int64_t* n_dev, int max_keys, float* out,
                        int32_t* nonfinite, cudaStream_t st) {
    const int sm = mlp_smem_bytes(P.field);
    const int64_t b3 = P.geom.b * P.geom.b * P.geom.b;
    const int gdec = grid_for((int64_t)max_keys * b3, 128, 8);
    if (P.field.kind == 0 && inr_is_default(P.field)) {
        // the default INR decodes on the tensor cores (tcgen05, decode_tc.cu)
        inr_bricks_tc_dev(P.field, P.geom, keys, n_dev, max_keys, out, nonfinite, st);
    } else {
        CINR_DISPATCH_INR(P.field, k_decode_bricks_dev, gdec, 128, sm, st, P.field, P.geom, keys, n_dev, max_keys, out,
                          nonfinite);
    }
}

static void maint_decode(const VcbMaintParams& P, const MaintWs& w, cudaStream_t st) {
    decode_keys(P, P.staged_keys, (const int64_t*)w.n_dec(), P.max_requests, P.staging, w.nonfinite, st);
    k_post_decode<<<1, 1, 0, st>>>(P, w);
}

// ---- brick-decode sharing across ranks (SURVEY §8e "optional brick sharing"): every
// rank's batch keys are all-gathered; each unique key is decoded once, by its owner
// rank (splitmix64(key) % world), into that owner's slab; the slabs are all-gathered
// and each rank copies its batch's bricks into its staging slab.  A key an owner cannot
// fit (more than `cap` owned keys) is decoded by every rank that needs it.  The decoder
// is deterministic per key, so staging equals the unshared decode bit for bit.
__device__ __forceinline__ int share_owner(long long key, int world) {
    return (int)(splitmix64((u64)key) % (u64)world);
}

// [n_dec, staged_keys[0..mr)] of this maintenance (n_dec = 0 when it was skipped)
__global__ void k_share_keys(VcbMaintParams P, MaintWs w, long long* out) {
    const long long n = *w.n_dec();
    for (int i = threadIdx.x; i <= P.max_requests; i += blockDim.x)
        out[i] = i == 0 ? n : (i - 1 < n ? P.staged_keys[i - 1] : -1);
}

// One CTA.  all: world rows of `stride` = mr + 1 ([n, keys...]).  Quadratic in the
// gathered keys (world * mr): a few hundred at the default batch.
__global__ void __launch_bounds__(1024) k_share_plan(const long long* all, int world, int rank, int stride, int cap,
                                                     long long* own, long long* counts, int32_t* src,
                                                     long long* ovf_keys, int32_t* ovf_idx) {
    extern __shared__ long long sk[];  // [M] keys (-1: none), then [M] owner of a first occurrence (-1: none)
    const int mr = stride - 1, M = world * mr;
    int* so = reinterpret_cast<int*>(sk + M);
    __shared__ int n_own, n_ovf;
    if (threadIdx.x == 0) n_own = n_ovf = 0;
    for (int t = threadIdx.x; t < M; t += blockDim.x) {
        const int q = t / mr, i = t - q * mr;
        sk[t] = i < all[(long long)q * stride] ? all[(long long)q * stride + 1 + i] : -1;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < M; t += blockDim.x) {
        const long long k = sk[t];
        bool first = k >= 0;
        for (int u = 0; u < t && first; u++) first = sk[u] != k;
        so[t] = first ? share_owner(k, world) : -1;
    }
    __syncthreads();
    // slot of a key = its rank among the distinct keys its owner holds
    auto slot_of = [&](long long k, int o) {
        int s = 0;
        for (int u = 0; u < M; u++) s += (so[u] == o && sk[u] < k);
        return s;
    };
    for (int t = threadIdx.x; t < M; t += blockDim.x) {
        const long long k = sk[t];
        if (so[t] != rank) continue;
        const int s = slot_of(k, rank);
        if (s < cap) {
            own[s] = k;
            atomicAdd(&n_own, 1);
        }
    }
    const long long n_mine = all[(long long)rank * stride];
    for (int i = threadIdx.x; i < mr; i += blockDim.x) {
        if (i >= n_mine) {
            src[i] = -1;
            continue;
        }
        const long long k = sk[rank * mr + i];
        const int o = share_owner(k, world);
        const int s = slot_of(k, o);
        if (s < cap) {
            src[i] = o * cap + s;
        } else {
            src[i] = -1;
            const int j = atomicAdd(&n_ovf, 1);
            ovf_keys[j] = k;
            ovf_idx[j] = i;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        counts[0] = n_own;
        counts[1] = n_ovf;
    }
}

// staging[i] <- gathered slab brick src[i] (or the locally decoded overflow brick);
// the decode-failure flag of the bricks this rank uses feeds k_post_decode
__global__ void k_share_scatter(VcbMaintParams P, MaintWs w, const float* gathered, const int32_t* flags, int cap,
                                const int32_t* src, const float* ovf_out, const int32_t* ovf_idx,
                                const long long* counts, const int32_t* ovf_flag) {
    const long long b3 = P.geom.b * P.geom.b * P.geom.b;
    const long long n = *w.n_dec(), n_ovf = counts[1];
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * b3; t += stride) {
        const long long i = t / b3, e = t - i * b3;
        const int s = src[i];
        if (s >= 0) P.staging[t] = gathered[(long long)s * b3 + e];
    }
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_ovf * b3; t += stride) {
        const long long j = t / b3, e = t - j * b3;
        P.staging[(long long)ovf_idx[j] * b3 + e] = ovf_out[t];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int bad = n_ovf > 0 && *ovf_flag != 0;
        for (long long i = 0; i < n && !bad; i++)
            if (src[i] >= 0 && flags[src[i] / cap]) bad = 1;
        if (bad) w.nonfinite[0] = 1;
    }
}

static int32_t maint_enqueue(const VcbMaintParams& P, cudaStream_t st) {
    if (P.max_requests < 1) return set_error("maintenance: batch size must be >= 1");
    if (P.max_requests > kMaxSel) return set_error("maintenance: max_requests > %d unsupported", kMaxSel);
    MaintWs w;
    int64_t need = maint_ws_layout(P.total, P.workspace, &w);
    if (need > P.workspace_bytes) return set_error("maintenance: workspace too small");
    // the decode flag is per maintenance (set by this call's decode, read by k_post_decode);
    // the workspace comes uninitialised from the caller.  The gate also reads the frame's
    // non-finite flag: a failed frame skips every step below on the device.
    k_maint_gate<<<1, 1, 0, st>>>(P, w);
    const int g = grid_for(P.total, 256, 8);
    // 1. drain miss reports into the request table (session.py:135-136)
    k_report<<<g, 256, 0, st>>>(P, w);
    // 2. collect: insert last dispatch's bricks (session.py:137-140)
    k_insert<<<1, kSelThreads, 0, st>>>(P, w);
    // 3. dispatch: select the batch (session.py:141, scheduler.py:152-169)
    k_pending<<<g, 256, 0, st>>>(P, w);
    k_select<<<1, kSelThreads, 0, st>>>(P, w);
    // 4. fulfill into the staging slab (inserted at the next maintenance); deferred: the
    //    caller runs vcb_maint_decode on its decode stream
    if (!P.defer_decode) maint_decode(P, w, st);
    g_launches += P.defer_decode ? 5 : 7;
    return check_launch("maintenance");
}

extern "C" int32_t vcb_maintenance(const VcbMaintParams* pp, void* stream_) {
    return maint_enqueue(*pp, (cudaStream_t)stream_);
}

// The maintenance as one CUDA graph: captured once per static configuration, then
// replayed each frame with session_frame updated in the kernels that take the
// maintenance parameters (the decode's arguments do not depend on the frame).
struct MaintGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaGraphNode_t> nodes;
    std::vector<cudaKernelNodeParams> kp;
    MaintWs w;
    long long launches = 0;
};

static bool takes_maint_params(const void* fn) {
    return fn == (const void*)k_maint_gate || fn == (const void*)k_report || fn == (const void*)k_insert ||
           fn == (const void*)k_pending || fn == (const void*)k_select || fn == (const void*)k_post_decode;
}

static void maint_graph_free(MaintGraph* g) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

extern "C" int32_t vcb_maint_graph_create(const VcbMaintParams* pp, void** out) {
    *out = nullptr;
    const VcbMaintParams& P = *pp;
    MaintGraph* g = new MaintGraph();
    if (maint_ws_layout(P.total, P.workspace, &g->w) > P.workspace_bytes) {
        delete g;
        return set_error("maint_graph: workspace too small");
    }
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
        delete g;
        return check_launch("maint_graph stream");
    }
    const long long before = g_launches;
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    const int32_t rc = maint_enqueue(P, cs);
    const cudaError_t e = cudaStreamEndCapture(cs, &g->graph);
    cudaStreamDestroy(cs);
    g->launches = g_launches - before;
    g_launches = before;
    if (rc != 0 || e != cudaSuccess) {
        maint_graph_free(g);
        return rc != 0 ? rc : set_error("maint_graph: capture failed: %s", cudaGetErrorString(e));
    }
    size_t n = 0;
    cudaGraphGetNodes(g->graph, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(g->graph, nodes.data(), &n);
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp;
        cudaGraphKernelNodeGetParams(nd, &kp);
        if (!takes_maint_params(kp.func)) continue;
        g->nodes.push_back(nd);
        g->kp.push_back(kp);
    }
    const size_t want = P.defer_decode ? 5 : 6;
    if (g->nodes.size() != want) {
        maint_graph_free(g);
        return set_error("maint_graph: %zu parameterised kernels captured, expected %zu", g->nodes.size(), want);
    }
    if (cudaGraphInstantiate(&g->exec, g->graph, 0) != cudaSuccess) {
        maint_graph_free(g);
        return check_launch("maint_graph instantiate");
    }
    *out = g;
    return 0;
}

extern "C" int32_t vcb_maint_graph_launch(void* handle, const VcbMaintParams* pp, void* stream_) {
    MaintGraph* g = (MaintGraph*)handle;
    if (!g) return set_error("maint_graph: null graph");
    VcbMaintParams P = *pp;  // kernel arguments are copied by SetParams
    void* args[2] = {&P, &g->w};
    for (size_t i = 0; i < g->nodes.size(); i++) {
        cudaKernelNodeParams kp = g->kp[i];
        kp.kernelParams = args;
        kp.extra = nullptr;
        if (cudaGraphExecKernelNodeSetParams(g->exec, g->nodes[i], &kp) != cudaSuccess)
            return check_launch("maint_graph set params");
    }
    cudaGraphLaunch(g->exec, (cudaStream_t)stream_);
    g_launches += g->launches;
    return check_launch("maint_graph launch");
}

extern "C" void vcb_maint_graph_destroy(void* handle) {
    if (handle) maint_graph_free((MaintGraph*)handle);
}

extern "C" int32_t vcb_share_keys(const VcbMaintParams* pp, int64_t* out, void* stream_) {
    const VcbMaintParams& P = *pp;
    MaintWs w;
    if (maint_ws_layout(P.total, P.workspace, &w) > P.workspace_bytes) return set_error("share_keys: workspace");
    k_share_keys<<<1, 256, 0, (cudaStream_t)stream_>>>(P, w, (long long*)out);
    return check_launch("share_keys");
}

extern "C" int32_t vcb_share_plan(const int64_t* all_keys, int32_t world, int32_t rank, int32_t max_requests,
                                  int32_t cap, int64_t* own_keys, int64_t* counts, int32_t* src, int64_t* ovf_keys,
                                  int32_t* ovf_idx, void* stream_) {
    const int M = world * max_requests;
    const size_t smem = (size_t)M * 12;
    if (world < 1 || rank < 0 || rank >= world || max_requests < 1 || cap < 1 || smem > 200 * 1024)
        return set_error("share_plan: world %d rank %d batch %d cap %d", world, rank, max_requests, cap);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_share_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_share_plan<<<1, 1024, smem, (cudaStream_t)stream_>>>((const long long*)all_keys, world, rank, max_requests + 1,
                                                            cap, (long long*)own_keys, (long long*)counts, src,
                                                            (long long*)ovf_keys, ovf_idx);
    return check_launch("share_plan");
}

extern "C" int32_t vcb_share_decode(const VcbMaintParams* pp, const int64_t* keys, const int64_t* n_keys,
                                    int32_t max_keys, float* out, int32_t* nonfinite, void* stream_) {
    decode_keys(*pp, keys, n_keys, max_keys, out, nonfinite, (cudaStream_t)stream_);
    g_launches += 1;
    return check_launch("share_decode");
}

extern "C" int32_t vcb_share_scatter(const VcbMaintParams* pp, const float* gathered, const int32_t* flags,
                                     int32_t cap, const int32_t* src, const float* ovf_out, const int32_t* ovf_idx,
                                     const int64_t* counts, const int32_t* ovf_flag, void* stream_) {
    const VcbMaintParams& P = *pp;
    MaintWs w;
    if (maint_ws_layout(P.total, P.workspace, &w) > P.workspace_bytes) return set_error("share_scatter: workspace");
    cudaStream_t st = (cudaStream_t)stream_;
    const int64_t b3 = P.geom.b * P.geom.b * P.geom.b;
    k_share_scatter<<<grid_for((int64_t)P.max_requests * b3, 256, 4), 256, 0, st>>>(
        P, w, gathered, flags, cap, src, ovf_out, ovf_idx, (const long long*)counts, ovf_flag);
    k_post_decode<<<1, 1, 0, st>>>(P, w);
    g_launches += 2;
    return check_launch("share_scatter");
}

extern "C" int32_t vcb_maint_decode(const VcbMaintParams* pp, void* stream_) {
    const VcbMaintParams& P = *pp;
    MaintWs w;
    int64_t need = maint_ws_layout(P.total, P.workspace, &w);
    if (need > P.workspace_bytes) return set_error("maint_decode: workspace too small");
    maint_decode(P, w, (cudaStream_t)stream_);
    g_launches += 2;
    return check_launch("maint_decode");
}
