// Field decoders: brick fill straight into a pool/staging slab, point batches
// (true misses / Field.sample_batch) and the macro-cell min/max pre-pass.
//
// Brick decode (scheduler.py:127-134 fulfill -> brickmath.py:125-139): sample s
// of a brick is x + B*(y + B*z) (x-fastest == pool [slot,z,y,x], P15); native =
// clip(origin + (x,y,z)*2^L, 0, V-1), normalized = (native + 0.5)/V in f64.
#include "common.cuh"
#include "fields.cuh"
#include "util.cuh"

namespace cinr {

__device__ __forceinline__ long long brick_origin(long long idx, long long b, int lod) {
    long long o = idx * (b << lod);
    return idx > 0 ? o - 1 : o;
}

template <int kInr>
__global__ void k_field_bricks(VcbField F, VcbBrickGeom G, int64_t n_keys, const int64_t* __restrict__ keys,
                               float* __restrict__ out, int32_t* nonfinite) {
    extern __shared__ __align__(16) float smem[];
    MlpSmem m;
    if (F.kind == 0) {
        stage_mlp(F, smem, m);
        __syncthreads();
    }
    const long long b = G.b, b3 = b * b * b;
    const long long total = n_keys * b3;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long ki = t / b3, s = t - ki * b3;
        const long long flat = keys[ki];
        int lod = 0;
        while (lod + 1 < G.n_lod && flat >= G.offset[lod + 1]) lod++;
        const long long lin = flat - G.offset[lod];
        const long long gx = G.grid[lod][0], gy = G.grid[lod][1];
        const long long ix = lin % gx, iy = (lin / gx) % gy, iz = lin / (gx * gy);
        const long long x = s % b, y = (s / b) % b, z = s / (b * b);
        long long nx = brick_origin(ix, b, lod) + (x << lod);
        long long ny = brick_origin(iy, b, lod) + (y << lod);
        long long nz = brick_origin(iz, b, lod) + (z << lod);
        nx = nx < G.dims[0] - 1 ? nx : G.dims[0] - 1;
        ny = ny < G.dims[1] - 1 ? ny : G.dims[1] - 1;
        nz = nz < G.dims[2] - 1 ? nz : G.dims[2] - 1;
        const double px = ((double)nx + 0.5) / (double)G.dims[0];
        const double py = ((double)ny + 0.5) / (double)G.dims[1];
        const double pz = ((double)nz + 0.5) / (double)G.dims[2];
        int bad = 0;
        out[t] = field_eval<kInr>(F, px, py, pz, m, &bad);
        if (bad) *nonfinite = 1;
    }
}

template <int kInr>
__global__ void k_field_points(VcbField F, int64_t n, const double* __restrict__ pos, float* __restrict__ out,
                               int32_t* nonfinite) {
    extern __shared__ __align__(16) float smem[];
    MlpSmem m;
    if (F.kind == 0) {
        stage_mlp(F, smem, m);
        __syncthreads();
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int bad = 0;
        out[i] = field_eval<kInr>(F, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], m, &bad);
        if (bad) *nonfinite = 1;
    }
}

// macrocell.py:49-74: lattice values at voxel centres ((i+0.5)/V), per cell the
// min/max over the cell dilated by one voxel.  One CTA per cell; the lattice is
// decoded on the fly (never materialised: 4096^3 would be 275 GB).
template <int kInr>
__global__ void k_macro_minmax(VcbField F, long long vx, long long vy, long long vz, long long cell, long long gx,
                               long long gy, long long gz, float* vmin, float* vmax) {
    extern __shared__ __align__(16) float smem[];
    __shared__ float rmin[32], rmax[32];
    MlpSmem m;
    if (F.kind == 0) {
        stage_mlp(F, smem, m);
        __syncthreads();
    }
    for (long long c = blockIdx.x; c < gx * gy * gz; c += gridDim.x) {
        const long long ci = c % gx, cj = (c / gx) % gy, ck = c / (gx * gy);
        const long long x0 = ci * cell - 1 > 0 ? ci * cell - 1 : 0, x1 = (ci + 1) * cell + 1 < vx ? (ci + 1) * cell + 1 : vx;
        const long long y0 = cj * cell - 1 > 0 ? cj * cell - 1 : 0, y1 = (cj + 1) * cell + 1 < vy ? (cj + 1) * cell + 1 : vy;
        const long long z0 = ck * cell - 1 > 0 ? ck * cell - 1 : 0, z1 = (ck + 1) * cell + 1 < vz ? (ck + 1) * cell + 1 : vz;
        const long long nx = x1 - x0, ny = y1 - y0, nz = z1 - z0, cnt = nx * ny * nz;
        float lo = INFINITY, hi = -INFINITY;
        for (long long t = threadIdx.x; t < cnt; t += blockDim.x) {
            const long long x = x0 + t % nx, y = y0 + (t / nx) % ny, z = z0 + t / (nx * ny);
            float v;
            if (F.kind == 1) {
                v = __ldg(F.lattice + (z * vy + y) * vx + x);
            } else {
                v = field_eval<kInr>(F, ((double)x + 0.5) / (double)vx, ((double)y + 0.5) / (double)vy,
                                      ((double)z + 0.5) / (double)vz, m, nullptr);
            }
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if ((threadIdx.x & 31) == 0) {
            rmin[threadIdx.x >> 5] = lo;
            rmax[threadIdx.x >> 5] = hi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < (int)(blockDim.x >> 5); i++) {
                lo = fminf(lo, rmin[i]);
                hi = fmaxf(hi, rmax[i]);
            }
            vmin[c] = lo;
            vmax[c] = hi;
        }
        __syncthreads();
    }
}

int mlp_smem_bytes(const VcbField& F) {
    if (F.kind != 0) return 0;
    int nw = 0, nb = 0;
    for (int L = 0; L < F.n_layers; L++) {
        nw += F.widths[L] * F.widths[L + 1];
        nb += F.widths[L + 1];
    }
    return (nw + nb) * (int)sizeof(float);
}


}  // namespace cinr

using namespace cinr;

extern "C" int32_t vcb_field_points(const VcbField* f, int64_t n, const double* pos, float* out, int32_t* nonfinite,
                                    void* stream) {
    if (n <= 0) return 0;
    const int sm = mlp_smem_bytes(*f);
    const int g = grid_for(n, 128, 8);
    CINR_DISPATCH_INR(*f, k_field_points, g, 128, sm, (cudaStream_t)stream, *f, n, pos, out, nonfinite);
    return check_launch("field_points");
}

extern "C" int32_t vcb_field_bricks(const VcbField* f, const VcbBrickGeom* g, int64_t n_keys, const int64_t* keys,
                                    float* out, int32_t* nonfinite, void* stream) {
    if (n_keys <= 0) return 0;
    const int sm = mlp_smem_bytes(*f);
    const int64_t total = n_keys * g->b * g->b * g->b;
    const int gr = grid_for(total, 128, 8);
    CINR_DISPATCH_INR(*f, k_field_bricks, gr, 128, sm, (cudaStream_t)stream, *f, *g, n_keys, keys, out, nonfinite);
    return check_launch("field_bricks");
}

extern "C" int32_t vcb_macro_minmax(const VcbField* f, const int64_t* dims, int64_t cell, float* vmin, float* vmax,
                                    void* stream) {
    const long long gx = (dims[0] + cell - 1) / cell, gy = (dims[1] + cell - 1) / cell, gz = (dims[2] + cell - 1) / cell;
    const int sm = mlp_smem_bytes(*f);
    long long cells = gx * gy * gz;
    int grid = (int)(cells < (long long)device_sms() * 16 ? cells : (long long)device_sms() * 16);
    CINR_DISPATCH_INR(*f, k_macro_minmax, grid, 256, sm, (cudaStream_t)stream, *f, dims[0], dims[1], dims[2], cell, gx,
                      gy, gz, vmin, vmax);
    return check_launch("macro_minmax");
}

// macrocell.py:120-128 update_majorants: mu(cell) = max of the TF's binned opacity
// maxima over bins [int(vmin*256), int(vmax*256)] (clamped), as f32.  The bins are
// the reference's f64 opacity_bin_maxima (host, 256 values); a range max does not
// depend on how the range is split, so this equals the reference's sparse-table
// query bit for bit.  Runs on every TF change (16.8 M cells at 4096^3).
namespace cinr {
__global__ void k_update_majorants(const float* __restrict__ vmin, const float* __restrict__ vmax, int64_t n,
                                   const double* __restrict__ bin_max, int bins, float* __restrict__ mu) {
    __shared__ double tab[9][256];  // tab[k][i] = max over bins [i, i + 2^k)
    for (int i = threadIdx.x; i < bins; i += blockDim.x) tab[0][i] = bin_max[i];
    __syncthreads();
    int levels = 1;
    for (int k = 1; (1 << k) <= bins && k < 9; k++) {
        const int h = 1 << (k - 1);
        for (int i = threadIdx.x; i + (1 << k) <= bins; i += blockDim.x) tab[k][i] = fmax(tab[k - 1][i], tab[k - 1][i + h]);
        __syncthreads();
        levels = k + 1;
    }
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        // (value * bins) in f32 is exact for bins = 2^8; astype(int64) truncates
        long long lo = (long long)(vmin[c] * (float)bins), hi = (long long)(vmax[c] * (float)bins);
        lo = lo < 0 ? 0 : (lo > bins - 1 ? bins - 1 : lo);
        hi = hi < 0 ? 0 : (hi > bins - 1 ? bins - 1 : hi);
        if (hi < lo) hi = lo;
        const int w = (int)(hi - lo + 1);
        int k = 31 - __clz(w);
        if (k > levels - 1) k = levels - 1;
        mu[c] = (float)fmax(tab[k][lo], tab[k][hi - (1 << k) + 1]);
    }
}
}  // namespace cinr

extern "C" int32_t vcb_update_majorants(const float* vmin, const float* vmax, int64_t n, const double* bin_max,
                                        int32_t bins, float* mu, void* stream) {
    if (n <= 0) return 0;
    if (bins < 1 || bins > 256) return cinr::set_error("update_majorants: bins must be in [1, 256]");
    cinr::k_update_majorants<<<cinr::grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(vmin, vmax, n, bin_max, bins,
                                                                                         mu);
    return cinr::check_launch("update_majorants");
}

// image_io.py:14-21 to_rgba8: (clip(f64(x), 0, 1) * 255 + 0.5).astype(uint8), per channel,
// on the device so a streamed frame leaves the GPU as 4 bytes per pixel.
namespace cinr {
__global__ void k_frame_rgba8(const float4* __restrict__ img, int64_t n, uchar4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = img[i];
        auto q = [](float x) -> unsigned char {
            double d = (double)x;
            d = d < 0.0 ? 0.0 : (d > 1.0 ? 1.0 : d);
            return (unsigned char)(int)__dadd_rn(__dmul_rn(d, 255.0), 0.5);
        };
        out[i] = make_uchar4(q(v.x), q(v.y), q(v.z), q(v.w));
    }
}
}  // namespace cinr

extern "C" int32_t vcb_frame_rgba8(const float* image, int64_t n_pixels, uint8_t* out, void* stream) {
    if (n_pixels <= 0) return 0;
    cinr::k_frame_rgba8<<<cinr::grid_for(n_pixels, 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4*>(image), n_pixels, reinterpret_cast<uchar4*>(out));
    return cinr::check_launch("frame_rgba8");
}
