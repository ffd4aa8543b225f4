// vr_quality.cu -- image metrics for step-size studies:
// quality.py:37-79 psnr / ssim on the rendered uint8 frames where they lie in
// HBM, so convergence_study never downloads its renders.
//
// PSNR: the sum of squared RGB differences is accumulated exactly in integers
// (the reference's float64 mean of integer squares is exact too, so the host's
// sse / n equals np.mean bit for bit).  SSIM: Rec. 601 luma, 11x11 Gaussian
// (sigma 1.5) windows over the valid region, the reference's constants and
// formula in float64; the window sums run in a different order than scipy's
// convolve2d, so SSIM agrees to ~1e-15 rather than bit for bit.
#include <cstdint>

#include "vr_common.cuh"

namespace vr {
namespace {

constexpr int kQBlock = 256;
constexpr int kWin = 11;
constexpr int kTile = 16;  // outputs per CTA side
constexpr int kHalo = kTile + kWin - 1;

__device__ unsigned long long warp_sum_u64(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kQBlock) sse_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b,
                                                      long long npix, int ca, int cb, unsigned long long *sse) {
    unsigned long long s = 0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npix; p += (long long)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int d = (int)__ldg(a + p * ca + c) - (int)__ldg(b + p * cb + c);
            s += (unsigned long long)(d * d);
        }
    }
    s = warp_sum_u64(s);
    __shared__ unsigned long long part[kQBlock / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kQBlock / 32; ++w) t += part[w];
        if (t) atomicAdd(sse, t);
    }
}

// quality.py:46-47
__device__ double luma(const uint8_t *p) {
    return (0.299 * (double)p[0] + 0.587 * (double)p[1]) + 0.114 * (double)p[2];
}

// One CTA = 16x16 outputs of the valid region; partial[cta] = sum of the
// per-pixel SSIM map over its outputs (reduced in a fixed order, so the
// result is deterministic).
__global__ void __launch_bounds__(kTile *kTile) ssim_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b,
                                                           int h, int w, int ca, int cb, const double *__restrict__ win,
                                                           double *partial) {
    __shared__ double lx[kHalo][kHalo + 1], ly[kHalo][kHalo + 1];
    __shared__ double wv[kWin * kWin];
    __shared__ double red[kTile * kTile];
    const int oh = h - kWin + 1, ow = w - kWin + 1;
    const int y0 = blockIdx.y * kTile, x0 = blockIdx.x * kTile;
    const int tid = threadIdx.y * kTile + threadIdx.x;
    for (int i = tid; i < kWin * kWin; i += kTile * kTile) wv[i] = win[i];
    for (int i = tid; i < kHalo * kHalo; i += kTile * kTile) {
        const int yy = y0 + i / kHalo, xx = x0 + i % kHalo;
        double vx = 0.0, vy = 0.0;
        if (yy < h && xx < w) {
            vx = luma(a + ((long long)yy * w + xx) * ca);
            vy = luma(b + ((long long)yy * w + xx) * cb);
        }
        lx[i / kHalo][i % kHalo] = vx;
        ly[i / kHalo][i % kHalo] = vy;
    }
    __syncthreads();
    const int oy = y0 + threadIdx.y, ox = x0 + threadIdx.x;
    double v = 0.0;
    if (oy < oh && ox < ow) {
        // convolve2d(..., mode="valid"): out[i,j] = sum_mn x[i+m, j+n] * win[10-m, 10-n]
        double mx = 0.0, my = 0.0, sxx = 0.0, syy = 0.0, sxy = 0.0;
        for (int m = 0; m < kWin; ++m) {
#pragma unroll
            for (int n = 0; n < kWin; ++n) {
                const double k = wv[(kWin - 1 - m) * kWin + (kWin - 1 - n)];
                const double x = lx[threadIdx.y + m][threadIdx.x + n];
                const double y = ly[threadIdx.y + m][threadIdx.x + n];
                mx += x * k;
                my += y * k;
                sxx += (x * x) * k;
                syy += (y * y) * k;
                sxy += (x * y) * k;
            }
        }
        // quality.py:72-78
        const double c1 = (0.01 * 255.0) * (0.01 * 255.0), c2 = (0.03 * 255.0) * (0.03 * 255.0);
        const double var_x = sxx - mx * mx, var_y = syy - my * my, cov = sxy - mx * my;
        const double num = ((2.0 * mx) * my + c1) * (2.0 * cov + c2);
        const double den = ((mx * mx + my * my) + c1) * ((var_x + var_y) + c2);
        v = num / den;
    }
    red[tid] = v;
    __syncthreads();
    for (int s = kTile * kTile / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    if (tid == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

// fixed-order sum of the CTA partials
__global__ void __launch_bounds__(kQBlock) sum_kernel(const double *partial, int n, double *out) {
    __shared__ double red[kQBlock];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += kQBlock) s += partial[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int k = kQBlock / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

cudaError_t launch_image_sse(const uint8_t *a, const uint8_t *b, long long npix, int ca, int cb,
                             unsigned long long *sse, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    long long g = (npix + kQBlock - 1) / kQBlock;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    sse_kernel<<<(int)g, kQBlock, 0, s>>>(a, b, npix, ca, cb, sse);
    return cudaGetLastError();
}

size_t image_ssim_scratch(int h, int w) {
    const int oh = h - kWin + 1, ow = w - kWin + 1;
    const size_t gx = (ow + kTile - 1) / kTile, gy = (oh + kTile - 1) / kTile;
    return sizeof(double) * (kWin * kWin + gx * gy);
}

cudaError_t launch_image_ssim(const uint8_t *a, const uint8_t *b, int h, int w, int ca, int cb, const double *win_host,
                              void *scratch, double *out_sum, cudaStream_t s) {
    const int oh = h - kWin + 1, ow = w - kWin + 1;
    dim3 grid((ow + kTile - 1) / kTile, (oh + kTile - 1) / kTile);
    double *win = static_cast<double *>(scratch);
    double *partial = win + kWin * kWin;
    cudaError_t e = cudaMemcpyAsync(win, win_host, sizeof(double) * kWin * kWin, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    ssim_kernel<<<grid, dim3(kTile, kTile), 0, s>>>(a, b, h, w, ca, cb, win, partial);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    sum_kernel<<<1, kQBlock, 0, s>>>(partial, (int)(grid.x * grid.y), out_sum);
    return cudaGetLastError();
}

}  // namespace vr
