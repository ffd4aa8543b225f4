// vr_prep.cu -- K1/K2/K4 kernels and the point sampler (see vr_prep.cuh).
#include <cstdlib>
#include <cfloat>
#include <climits>

#include "vr_prep.cuh"

namespace vr {
namespace {

constexpr int kBlock = 256;

VR_D int warp_min(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
VR_D int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
VR_D unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// grid of a grid-stride kernel: one thread per item, at most `per_sm` CTAs per SM
int grid_for(long long n, int block, int per_sm = 16) {
    const long long cap = (long long)device_sms() * per_sm;
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

// ------------------------------------------------------------ value range

__global__ void init_minmax_kernel(int *out, int count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        out[2 * i] = INT_MAX;
        out[2 * i + 1] = INT_MIN;
    }
}

__global__ void __launch_bounds__(kBlock) value_range_kernel(const int16_t *__restrict__ v, long long n, int *out) {
    int lo = INT_MAX, hi = INT_MIN;
    long long nvec = n / 8;
    const int4 *v8 = reinterpret_cast<const int4 *>(v);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
        int4 q = __ldg(v8 + i);
        const int16_t *h = reinterpret_cast<const int16_t *>(&q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            lo = min(lo, (int)h[k]);
            hi = max(hi, (int)h[k]);
        }
    }
    for (long long i = nvec * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        lo = min(lo, (int)v[i]);
        hi = max(hi, (int)v[i]);
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, lo);
        atomicMax(out + 1, hi);
    }
}

// --------------------------------------------------------------- phantoms

struct Ellipsoid {
    double cx, cy, cz, ax, ay, az, s_min, width;
};

struct PhantomArgs {
    int kind, nx, ny, nz;
    Ellipsoid e[4];       // torso: body, spine, blob_l, blob_r
    double c[3];          // sphere: integer centres d//2; shell: (d-1)/2
    double radius;        // sphere: min(dims)//2 ; shell: min(dims)/2
    double r_in, r_out;   // shell: 0.55*radius, 0.80*radius
};

// phantoms.py:32-42
VR_D double ellipsoid_blend(const Ellipsoid &E, double x, double y, double z) {
    double qx = (x - E.cx) / E.ax;
    double qy = (y - E.cy) / E.ay;
    double qz = (z - E.cz) / E.az;
    double e = sqrt((qx * qx + qy * qy) + qz * qz);
    double v = (1.0 - e) * E.s_min / E.width + 0.5;
    return fmin(fmax(v, 0.0), 1.0);
}

__global__ void __launch_bounds__(kBlock) phantom_kernel(const __grid_constant__ PhantomArgs p, int16_t *out) {
    long long n = (long long)p.nx * p.ny * p.nz;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int ix = (int)(i % p.nx);
        long long r = i / p.nx;
        int iy = (int)(r % p.ny);
        int iz = (int)(r / p.ny);
        double x = ix, y = iy, z = iz;
        double field;
        if (p.kind == 2) {  // torso, phantoms.py:63-79
            double body = ellipsoid_blend(p.e[0], x, y, z);
            double spine = ellipsoid_blend(p.e[1], x, y, z);
            double bl = ellipsoid_blend(p.e[2], x, y, z);
            double br = ellipsoid_blend(p.e[3], x, y, z);
            double bone = fmax(spine, fmax(bl, br));
            field = (-1000.0 + 1040.0 * body) + 1160.0 * bone;
        } else {
            double dx = x - p.c[0], dy = y - p.c[1], dz = z - p.c[2];
            double rr = sqrt((dx * dx + dy * dy) + dz * dz);
            if (p.kind == 0) {  // sphere, phantoms.py:45-50
                double v = 1000.0 - 2000.0 * rr / p.radius;
                field = fmin(fmax(v, -1000.0), 1000.0);
            } else {  // shell, phantoms.py:53-60
                double d = fmax(p.r_in - rr, rr - p.r_out);
                double band = fmin(fmax(0.5 - d / 1.5, 0.0), 1.0);
                field = -1000.0 + 1800.0 * band;
            }
        }
        out[i] = (int16_t)rint(field);
    }
}

// ------------------------------------------------------------- block minmax

VR_D void block_coords(const Layout &L, int b, int &bi, int &bj, int &bk) {
    bi = b % L.nb[0];
    int r = b / L.nb[0];
    bj = r % L.nb[1];
    bk = r / L.nb[1];
}

// one CTA per (block, z-chunk); rows of the block are read x-contiguous
__global__ void __launch_bounds__(kBlock) block_minmax_kernel(const int16_t *__restrict__ vol, const Layout L,
                                                              int *vmin, int *vmax) {
    int b = blockIdx.x;
    int bi, bj, bk;
    block_coords(L, b, bi, bj, bk);
    int ox = block_origin(L, bi), oy = block_origin(L, bj), oz = block_origin(L, bk);
    int ex = block_extent(L, 0, bi), ey = block_extent(L, 1, bj), ez = block_extent(L, 2, bk);
    int lo = INT_MAX, hi = INT_MIN;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // one z-slice per CTA row of the grid; each warp walks rows x-contiguously
    for (int z = blockIdx.y; z < ez; z += gridDim.y) {
        const int16_t *plane = vol + (long long)(oz + z) * L.pz + (long long)oy * L.py + ox;
        for (int y = wid; y < ey; y += nw) {
            const int16_t *row = plane + (long long)y * L.py;
            for (int x = lane; x < ex; x += 32) {
                int v = __ldg(row + x);
                lo = min(lo, v);
                hi = max(hi, v);
            }
        }
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0 && lo <= hi) {
        atomicMin(vmin + b, lo);
        atomicMax(vmax + b, hi);
    }
}

__global__ void init_block_minmax_kernel(int *vmin, int *vmax, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        vmin[i] = INT_MAX;
        vmax[i] = INT_MIN;
    }
}

// ------------------------------------------------------------- visibility

// transfer.py:120-125 ClassifiedLUT.bin_index
VR_D int classified_bin(double s, double lo, double bin_width, int nbins) {
    double f = floor((s - lo) / bin_width);
    if (f < 0.0) return 0;
    if (f > (double)(nbins - 1)) return nbins - 1;
    return (int)f;
}

// The same bin with the quotient estimated by a reciprocal multiply; the
// exact division only runs when the estimate lies within 1e-9 of an integer
// (the estimate is within a few ulp of the correctly rounded quotient).
VR_D int classified_bin_fast(double s, double lo, double bin_width, double inv_width, int nbins) {
    const double q = (s - lo) * inv_width;
    double f = floor(q);
    const double fr = q - f;
    if (fr < 1e-9 || fr > 1.0 - 1e-9) f = floor((s - lo) / bin_width);
    if (f < 0.0) return 0;
    if (f > (double)(nbins - 1)) return nbins - 1;
    return (int)f;
}

#ifndef VR_SETUP_THREADS
#define VR_SETUP_THREADS 1024
#endif
constexpr int kSetupThreads = VR_SETUP_THREADS;  // 64..1024 (2048 visbits words split evenly)
constexpr int kSetupWarps = kSetupThreads / 32;
static_assert(kSetupThreads >= 64 && kSetupThreads <= 1024 && 2048 % kSetupThreads == 0, "setup CTA size");

// cull_empty (blocks.py:161-173) + the per-value visibility bitmask that
// fit_bounding_box (blocks.py:176-199) tests per voxel, and the list of
// non-empty blocks the AABB fit walks.  One CTA.
__global__ void __launch_bounds__(kSetupThreads) vis_setup_kernel(const VisArgs v) {
    pdl_enter();
    extern __shared__ int prefix[];  // nbins + 1
    __shared__ int warp_tot[kSetupWarps];
    __shared__ unsigned int n_empty;
    __shared__ int n_list;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    zero_fill(v.zero);
    __shared__ int first_vis, last_vis;
    if (tid == 0) {
        first_vis = v.nbins;
        last_vis = -1;
    }
    // exclusive prefix over the bins with nonzero opacity
    // (ClassifiedLUT.opacity_prefix, transfer.py:131-133): block-wide scan
    const int per = (v.nbins + kSetupThreads - 1) / kSetupThreads;
    const int b0 = min(tid * per, v.nbins), b1 = min(b0 + per, v.nbins);
    int s = 0;
    for (int i = b0; i < b1; ++i) s += (__ldg(v.lut + 4 * i + 3) > 0.0) ? 1 : 0;
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    if (tid == 0) {
        n_empty = 0;
        n_list = 0;
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the warp totals
        const int w = lane < kSetupWarps ? warp_tot[lane] : 0;
        int inc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane < kSetupWarps) warp_tot[lane] = inc - w;
    }
    __syncthreads();
    int run = warp_tot[wid] + incl - s;
    for (int i = b0; i < b1; ++i) {
        prefix[i] = run;
        const int vis = (__ldg(v.lut + 4 * i + 3) > 0.0) ? 1 : 0;
        run += vis;
        if (vis && v.lut_range) {
            atomicMin(&first_vis, i);
            atomicMax(&last_vis, i);
        }
    }
    if (b1 == v.nbins && b0 < b1) prefix[v.nbins] = run;
    __syncthreads();
    // visible values before each visbits word (for the AABB fit's cell test)
    {
        constexpr int kWords = 2048 / kSetupThreads;  // visbits words per thread
        int cnt[kWords], sum = 0;
#pragma unroll
        for (int j = 0; j < kWords; ++j) {
            cnt[j] = __popc(v.visbits[kWords * tid + j]);
            sum += cnt[j];
        }
        int inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        __syncthreads();  // warp_tot reused
        if (lane == 31) warp_tot[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const int w = lane < kSetupWarps ? warp_tot[lane] : 0;
            int x = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane < kSetupWarps) warp_tot[lane] = x - w;
        }
        __syncthreads();
        int ex = warp_tot[wid] + inc - sum;
#pragma unroll
        for (int j = 0; j < kWords; ++j) {
            v.visprefix[kWords * tid + j] = ex;
            ex += cnt[j];
        }
        if (tid == kSetupThreads - 1) v.visprefix[2048] = ex;
    }
    const double inv_w = 1.0 / v.bin_width;
    // interval test per block, sentinel AABB for the fit kernel
    for (int b = tid; b < v.nblocks; b += kSetupThreads) {
        int lo = classified_bin_fast((double)v.vmin[b], v.lut_lo, v.bin_width, inv_w, v.nbins);
        int hi = classified_bin_fast((double)v.vmax[b], v.lut_lo, v.bin_width, inv_w, v.nbins);
        bool visible = (prefix[hi + 1] - prefix[lo]) > 0;
        v.empty[b] = visible ? 0 : 1;
        if (!visible)
            atomicAdd(&n_empty, 1u);
        else
            v.list[1 + atomicAdd(&n_list, 1)] = b;
        int *ab = v.aabb + 6 * b;
        ab[0] = ab[1] = ab[2] = INT_MAX;
        ab[3] = ab[4] = ab[5] = -1;
    }
    __syncthreads();
    int vlo = 0, vhi = 0;
    if (v.lut_range) block_value_range<kSetupThreads>(v.lut_lo, v.lut_inv_w, v.nbins, first_vis, last_vis, vlo, vhi);
    if (tid == 0) {
        v.counters[0] = n_empty;
        v.counters[1] = 0;
        v.list[0] = n_list;
        if (v.lut_range) {
            v.lut_range[0] = first_vis;
            v.lut_range[1] = last_vis;
            v.lut_range[2] = vlo;
            v.lut_range[3] = vhi;
        }
    }
    if (tid < 6) v.uni[tid] = tid < 3 ? INT_MAX : INT_MIN;
}

// Visibility bit per int16 value, lut.rgba[bin_index(v), 3] > 0 (the test
// fit_bounding_box applies per voxel): one warp per 32-value word, spread
// over the GPU (65536 bins on a single SM were 12 us of issue time).
__global__ void __launch_bounds__(kBlock) visbits_kernel(const VisArgs v) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= 2048) return;
    const double inv_w = 1.0 / v.bin_width;
    const int val = w * 32 + lane - 32768;
    const int bin = classified_bin_fast((double)val, v.lut_lo, v.bin_width, inv_w, v.nbins);
    const unsigned int bits = __ballot_sync(0xffffffffu, __ldg(v.lut + 4 * bin + 3) > 0.0);
    if (lane == 0) v.visbits[w] = bits;
}

// number of visible int16 values in [lo, hi]
VR_D int count_visible(const unsigned int *bits, const int *prefix, int lo, int hi) {
    const unsigned u0 = (unsigned)(lo + 32768), u1 = (unsigned)(hi + 32768);
    const unsigned w0 = u0 >> 5, w1 = u1 >> 5;
    const unsigned m0 = 0xffffffffu << (u0 & 31u), m1 = 0xffffffffu >> (31u - (u1 & 31u));
    if (w0 == w1) return __popc(bits[w0] & m0 & m1);
    return __popc(bits[w0] & m0) + __popc(bits[w1] & m1) + (prefix[w1] - prefix[w0 + 1]);
}

// fit_bounding_box (blocks.py:176-199): local min/max of visible voxels.
// Persistent: each CTA walks (non-empty block, 4-voxel z-layer of cells)
// items: the layer's cells whose value bound
// (the volume's 4^3 cell table, which covers every voxel value in the cell)
// holds a visible value are collected, then their voxels tested one per
// thread -- the other cells cannot hold a visible voxel.  Exact: the result is
// that of a full scan.
constexpr int kAabbThreads = 256;
constexpr int kCand = 1024;  // cells examined per pass
__global__ void __launch_bounds__(kAabbThreads) aabb_kernel(const int16_t *__restrict__ bricks, const Layout L,
                                                            const VisArgs v, int zmax) {
    pdl_enter();
    __shared__ unsigned int bits[2048];
    __shared__ int prefix[2049];
    __shared__ int cand[kCand];
    __shared__ int ncand;
    const int count = v.list[0];
    const int layers = (zmax + 3) / 4 + 1;  // cell layers a block can touch
    const long long items = (long long)count * layers;
    if ((long long)blockIdx.x >= items) return;  // before staging 16 KB for nothing
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) bits[i] = v.visbits[i];
    for (int i = threadIdx.x; i < 2049; i += blockDim.x) prefix[i] = v.visprefix[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int b = v.list[1 + (int)(it / layers)];
        int bi, bj, bk;
        block_coords(L, b, bi, bj, bk);
        const int ox = block_origin(L, bi), oy = block_origin(L, bj), oz = block_origin(L, bk);
        const int ex = block_extent(L, 0, bi), ey = block_extent(L, 1, bj), ez = block_extent(L, 2, bk);
        const int cz = (oz >> 2) + (int)(it % layers);
        if (cz > (oz + ez - 1) >> 2) continue;
        const int cx0 = ox >> 2, cx1 = (ox + ex - 1) >> 2, cy0 = oy >> 2, cy1 = (oy + ey - 1) >> 2;
        const int ncx = cx1 - cx0 + 1, ncells = ncx * (cy1 - cy0 + 1);
        if (v.mcells) {
            // the macro cells (16^3) over this cell layer: when none can hold a
            // visible value, neither can any of its cells.  Every warp takes the
            // same decision, so the CTA skips the item without a barrier.
            const int mx0 = cx0 >> 2, nmxi = (cx1 >> 2) - mx0 + 1, my0 = cy0 >> 2;
            const int nm = nmxi * ((cy1 >> 2) - my0 + 1);
            const short2 *mrow = v.mcells + (long long)(cz >> 2) * v.nmy * v.nmx;
            bool vis = false;
            for (int m = lane; m < nm && !vis; m += 32) {
                const short2 mb = __ldg(mrow + (long long)(my0 + m / nmxi) * v.nmx + mx0 + m % nmxi);
                vis = count_visible(bits, prefix, mb.x, mb.y) > 0;
            }
            if (!__any_sync(0xffffffffu, vis)) continue;
        }
        int mnx = INT_MAX, mny = INT_MAX, mnz = INT_MAX, mxx = -1, mxy = -1, mxz = -1;
        // in chunks of kCand cells: (1) collect the cells that may hold a
        // visible voxel, (2) test their voxels, one per thread
        for (int c0 = 0; c0 < ncells; c0 += kCand) {
            if (threadIdx.x == 0) ncand = 0;
            __syncthreads();
            // (loads of a pass issued before any is used: one memory round
            // trip per pass instead of one per iteration)
            const int cend = min(ncells, c0 + kCand);
            short2 cbs[kCand / kAabbThreads];
#pragma unroll
            for (int j = 0; j < kCand / kAabbThreads; ++j) {
                const int c = c0 + (int)threadIdx.x + j * kAabbThreads;
                if (c < cend)
                    cbs[j] = __ldg(v.cells + ((long long)cz * v.ncy + cy0 + c / ncx) * v.ncx + cx0 + c % ncx);
            }
#pragma unroll
            for (int j = 0; j < kCand / kAabbThreads; ++j) {
                const int c = c0 + (int)threadIdx.x + j * kAabbThreads;
                if (c >= cend) continue;
                const int cx = cx0 + c % ncx, cy = cy0 + c / ncx;
                const short2 cb = cbs[j];
                const int nv = count_visible(bits, prefix, cb.x, cb.y);
                if (nv == (int)cb.y - (int)cb.x + 1) {
                    // every value the cell can hold is visible: all its voxels
                    // in the block are, no scan needed
                    mnx = min(mnx, max(cx * 4, ox) - ox); mxx = max(mxx, min(cx * 4 + 3, ox + ex - 1) - ox);
                    mny = min(mny, max(cy * 4, oy) - oy); mxy = max(mxy, min(cy * 4 + 3, oy + ey - 1) - oy);
                    mnz = min(mnz, max(cz * 4, oz) - oz); mxz = max(mxz, min(cz * 4 + 3, oz + ez - 1) - oz);
                } else if (nv > 0) {
                    cand[atomicAdd(&ncand, 1)] = c;
                }
            }
            __syncthreads();
            // the candidate cells' voxels, 16 bytes (8 voxels: half a z-slice
            // of the brick) per thread and load, all loads of a pass in flight
            const int nvec = ncand * 8;
            constexpr int kU = 4;
            for (int e0 = threadIdx.x; e0 < nvec; e0 += kAabbThreads * kU) {
                uint4 val[kU];
#pragma unroll
                for (int j = 0; j < kU; ++j) {
                    const int e = e0 + j * kAabbThreads;
                    if (e < nvec) {
                        // a cell is one 4^3 brick: 128 contiguous bytes, x fastest
                        const int c = cand[e >> 3];
                        const long long brick = ((long long)cz * v.ncy + cy0 + c / ncx) * v.ncx + cx0 + c % ncx;
                        val[j] = __ldg(reinterpret_cast<const uint4 *>(bricks + brick * 64) + (e & 7));
                    }
                }
#pragma unroll
                for (int j = 0; j < kU; ++j) {
                    const int e = e0 + j * kAabbThreads;
                    if (e >= nvec) continue;
                    const int c = cand[e >> 3], q = e & 7;
                    const int z = cz * 4 + (q >> 1) - oz;
                    const int bx = (cx0 + c % ncx) * 4 - ox, by = (cy0 + c / ncx) * 4 - oy;
                    const unsigned words[4] = {val[j].x, val[j].y, val[j].z, val[j].w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        // voxel w = 8q + k of the brick: x = k & 3, y = (2q + k/4) & 3, z = q / 2
                        const int x = bx + (k & 3), y = by + (((q << 1) + (k >> 2)) & 3);
                        const unsigned u = (unsigned)((int)(short)(words[k >> 1] >> (16 * (k & 1))) + 32768);
                        if (x >= 0 && x < ex && y >= 0 && y < ey && z >= 0 && z < ez &&
                            ((bits[u >> 5] >> (u & 31)) & 1u)) {
                            mnx = min(mnx, x); mxx = max(mxx, x);
                            mny = min(mny, y); mxy = max(mxy, y);
                            mnz = min(mnz, z); mxz = max(mxz, z);
                        }
                    }
                }
            }
            __syncthreads();  // cand / ncand reused
        }
        mnx = warp_min(mnx); mny = warp_min(mny); mnz = warp_min(mnz);
        mxx = warp_max(mxx); mxy = warp_max(mxy); mxz = warp_max(mxz);
        if (lane == 0 && mxx >= 0) {
            int *ab = v.aabb + 6 * b;
            atomicMin(ab + 0, mnx); atomicMin(ab + 1, mny); atomicMin(ab + 2, mnz);
            atomicMax(ab + 3, mxx); atomicMax(ab + 4, mxy); atomicMax(ab + 5, mxz);
        }
    }
}

// dilate by one, clip to the block, globalise (blocks.py:189-198) and apply
// the render margin (render.py:388-390)
__global__ void box_kernel(const Layout L, const VisArgs v) {
    pdl_enter();
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= v.nblocks) return;
    int bi, bj, bk;
    block_coords(L, b, bi, bj, bk);
    const int org[3] = {block_origin(L, bi), block_origin(L, bj), block_origin(L, bk)};
    const int ext[3] = {block_extent(L, 0, bi), block_extent(L, 1, bj), block_extent(L, 2, bk)};
    const int *ab = v.aabb + 6 * b;
    bool fitted = !v.empty[b] && ab[3] >= 0;
    v.box[8 * b + 3] = v.empty[b] ? 1.0f : 0.0f;
    v.box[8 * b + 7] = 0.0f;
    if (!v.empty[b] && !fitted) atomicAdd(v.counters + 1, 1ull);  // reference raises EmptyBlock
    for (int k = 0; k < 3; ++k) {
        long long lo, hi;
        if (fitted) {
            lo = org[k] + max(ab[k] - 1, 0);
            hi = org[k] + min(ab[3 + k] + 1, ext[k] - 1);
        } else {
            lo = LLONG_MAX / 2;
            hi = -1;
        }
        // integers +- margin (2 or 3): exact in float32 for |value| < 2^24
        v.box[8 * b + k] = (float)((double)lo - v.margin);
        v.box[8 * b + 4 + k] = (float)((double)hi + v.margin);
        if (v.aabb_global) {
            v.aabb_global[6 * b + k] = lo;
            v.aabb_global[6 * b + 3 + k] = hi;
        }
        if (fitted) {
            atomicMin(v.uni + k, (int)lo);
            atomicMax(v.uni + 3 + k, (int)hi);
        }
    }
}

// ----------------------------------------------------------- K1 bricks

__global__ void __launch_bounds__(kBlock) brick_kernel(const int16_t *__restrict__ vol, int nx, int ny, int nz,
                                                       int bnx, int bny, long long total, int16_t *bricks) {
    long long py = nx, pz = (long long)nx * ny;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        long long b = e >> 6;
        int w = (int)(e & 63);
        int bx = (int)(b % bnx);
        long long r = b / bnx;
        int by = (int)(r % bny), bz = (int)(r / bny);
        int x = bx * 4 + (w & 3), y = by * 4 + ((w >> 2) & 3), z = bz * 4 + (w >> 4);
        bricks[e] = (x < nx && y < ny && z < nz) ? __ldg(vol + z * pz + y * py + x) : (int16_t)0;
    }
}

// ------------------------------------------------------- transparency culling

// ---------------------------------------------- interpolant bounds per cube
// Bounds of the Catmull-Rom (and trilinear) interpolant over each unit cube
// g = (gx, gy, gz) + [0,1)^3, i.e. of every sample whose base index is g,
// under any block-local clamping of its taps.  Separable and rigorous: along
// x each row of four taps (a, b, c, d) is a Catmull-Rom segment whose Bezier
// control points are b, b + (c-a)/6, c - (d-b)/6, c, so the segment lies in
// their hull (convex hull property); clamping replaces a by b or d by c, which
// adds two control points.  Along y (then z) the rows are intervals [L, H];
// since w0, w3 <= 0 <= w1, w2 on [0,1] the interpolant is at most the
// segment through (L0, H1, H2, L3) and at least the one through (H0, L1, L2,
// H3), bounded again by their hulls (clamping: L0 -> L1, L3 -> L2, ...).
// Trilinear values are convex combinations of the cube's corners, which the
// hulls contain.  Evaluated in float32 and rounded outwards by one unit.
struct Span {
    float lo, hi;
};

VR_D Span row_hull(float a, float b, float c, float d) {
    const float k = 1.0f / 6.0f;
    const float p1 = b + (c - a) * k, p1c = b + (c - b) * k;
    const float p2 = c - (d - b) * k, p2c = c - (c - b) * k;
    Span s;
    s.lo = fminf(fminf(fminf(b, c), fminf(p1, p1c)), fminf(p2, p2c));
    s.hi = fmaxf(fmaxf(fmaxf(b, c), fmaxf(p1, p1c)), fmaxf(p2, p2c));
    return s;
}

VR_D Span span_hull(Span s0, Span s1, Span s2, Span s3) {
    const float k = 1.0f / 6.0f;
    const float l0 = fminf(s0.lo, s1.lo), l3 = fminf(s3.lo, s2.lo);  // clamped variants
    const float h0 = fmaxf(s0.hi, s1.hi), h3 = fmaxf(s3.hi, s2.hi);
    Span r;
    r.hi = fmaxf(fmaxf(s1.hi, s2.hi), fmaxf(s1.hi + (s2.hi - l0) * k, s2.hi - (l3 - s1.hi) * k));
    r.lo = fminf(fminf(s1.lo, s2.lo), fminf(s1.lo + (s2.lo - h0) * k, s2.lo - (h3 - s1.lo) * k));
    return r;
}

constexpr int kCubeTile = 8;
constexpr int kCubeHalo = kCubeTile + 3;

// one CTA = 8^3 cubes; the taps [g-1, g+2] of the tile staged in shared memory
__global__ void __launch_bounds__(512) cube_bound_kernel(const int16_t *__restrict__ vol, int nx, int ny, int nz,
                                                         int bnx, int bny, short2 *__restrict__ cubes) {
    __shared__ float tile[kCubeHalo][kCubeHalo][kCubeHalo];
    const int x0 = blockIdx.x * kCubeTile, y0 = blockIdx.y * kCubeTile, z0 = blockIdx.z * kCubeTile;
    const long long py = nx, pz = (long long)nx * ny;
    for (int i = threadIdx.x; i < kCubeHalo * kCubeHalo * kCubeHalo; i += blockDim.x) {
        const int lx = i % kCubeHalo, ly = (i / kCubeHalo) % kCubeHalo, lz = i / (kCubeHalo * kCubeHalo);
        const int gx = min(max(x0 - 1 + lx, 0), nx - 1);
        const int gy = min(max(y0 - 1 + ly, 0), ny - 1);
        const int gz = min(max(z0 - 1 + lz, 0), nz - 1);
        tile[lz][ly][lx] = (float)__ldg(vol + gz * pz + gy * py + gx);
    }
    __syncthreads();
    const int cx = threadIdx.x & 7, cy = (threadIdx.x >> 3) & 7, cz = threadIdx.x >> 6;
    const int gx = x0 + cx, gy = y0 + cy, gz = z0 + cz;
    if (gx >= nx || gy >= ny || gz >= nz) return;
    Span planes[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        Span rows[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float *r = &tile[cz + k][cy + j][cx];
            rows[j] = row_hull(r[0], r[1], r[2], r[3]);
        }
        planes[k] = span_hull(rows[0], rows[1], rows[2], rows[3]);
    }
    const Span v = span_hull(planes[0], planes[1], planes[2], planes[3]);
    const float lo = fmaxf(floorf(v.lo) - 1.0f, -32768.0f), hi = fminf(ceilf(v.hi) + 1.0f, 32767.0f);
    const long long o = ((((long long)(gz >> 2) * bny + (gy >> 2)) * bnx + (gx >> 2)) << 6) + ((gz & 3) << 4) +
                        ((gy & 3) << 2) + (gx & 3);
    cubes[o] = make_short2((short)lo, (short)hi);
}

// cells[c] = union of the bounds of the cubes in the 4^3 cell c (= one brick
// of the cube table)
__global__ void __launch_bounds__(kBlock) cell_from_cubes_kernel(const short2 *__restrict__ cubes, int nx, int ny,
                                                                 int nz, int ncx, int ncy, int ncz, short2 *cells) {
    const long long n = (long long)ncx * ncy * ncz;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
        const int cx = (int)(c % ncx);
        const long long r = c / ncx;
        const int cy = (int)(r % ncy), cz = (int)(r / ncy);
        int lo = INT_MAX, hi = INT_MIN;
        for (int i = 0; i < 64; ++i) {
            const int x = cx * 4 + (i & 3), y = cy * 4 + ((i >> 2) & 3), z = cz * 4 + (i >> 4);
            if (x >= nx || y >= ny || z >= nz) continue;  // padding entries are never written
            const short2 b = __ldg(cubes + c * 64 + i);
            lo = min(lo, (int)b.x);
            hi = max(hi, (int)b.y);
        }
        cells[c] = make_short2((short)lo, (short)hi);
    }
}

__global__ void lut_range_kernel(const double *lut, int nbins, double lut_lo, double lut_inv_w, int *range,
                                 const ZeroSpec zero) {
    pdl_enter();
    __shared__ int first, last;
    zero_fill(zero);
    if (threadIdx.x == 0) {
        first = nbins;
        last = -1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) {
        if (__ldg(lut + 4 * i + 3) > 0.0) {
            atomicMin(&first, i);
            atomicMax(&last, i);
        }
    }
    __syncthreads();
    int vlo, vhi;
    block_value_range<kSetupThreads>(lut_lo, lut_inv_w, nbins, first, last, vlo, vhi);
    if (threadIdx.x == 0) {
        range[0] = first;
        range[1] = last;
        range[2] = vlo;
        range[3] = vhi;
    }
}

// one CTA per view: blocks_visited of view v into out[5 v + 2] (hits may be
// null: only the counters), the frame's visibility counters into [5 v + 3..4]
__global__ void count_hits_kernel(const uint8_t *hits, int n, unsigned long long *out,
                                  const unsigned long long *vis_counters) {
    pdl_enter();
    const long long v = blockIdx.x;
    out += 5 * v;
    if (threadIdx.x < 2) out[3 + threadIdx.x] = vis_counters ? vis_counters[threadIdx.x] : 0ull;
    if (!hits) return;
    hits += v * n;
    unsigned long long c = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) c += hits[i] ? 1 : 0;
    c = warp_sum(c);
    __shared__ unsigned long long part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
        out[2] = s;
    }
}

// ------------------------------------------- pre-integrated culling table
// nz[i * (n+1) + j] = number of table cells (front f < i, back b < j) with
// opacity > 0 (table (n, n, 4) float64, render.py:425): the square of bins
// [i0, i1)^2 is transparent iff its four-corner difference is 0.  One CTA:
// row prefixes, then column prefixes.
__global__ void tbl_nonzero_kernel(const double *table, int n, int *nz) {
    pdl_enter();
    const int w = n + 1;
    for (int i = threadIdx.x; i < w; i += blockDim.x) nz[i] = 0;  // row 0
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int run = 0;
        nz[(i + 1) * w] = 0;
        for (int j = 0; j < n; ++j) {
            run += __ldg(table + 4 * ((long long)i * n + j) + 3) > 0.0 ? 1 : 0;
            nz[(i + 1) * w + j + 1] = run;
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < w; j += blockDim.x)
        for (int i = 1; i < w; ++i) nz[i * w + j] += nz[(i - 1) * w + j];
}

// --------------------------------------------------------- preclassify

__global__ void __launch_bounds__(kBlock) preclassify_kernel(const int16_t *__restrict__ vol, long long n,
                                                             const double *__restrict__ lut, int nbins,
                                                             double lo, double bw, uint8_t *rgba) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int k = classified_bin((double)vol[i], lo, bw, nbins);
        // interleaved (nz, ny, nx, 4), the layout transfer.py:142-145 returns
        reinterpret_cast<uchar4 *>(rgba)[i] =
            make_uchar4((uint8_t)rint(__ldg(lut + 4 * k) * 255.0), (uint8_t)rint(__ldg(lut + 4 * k + 1) * 255.0),
                        (uint8_t)rint(__ldg(lut + 4 * k + 2) * 255.0), (uint8_t)rint(__ldg(lut + 4 * k + 3) * 255.0));
    }
}

// ------------------------------------------------------- point sampling

__global__ void __launch_bounds__(kBlock) sample_points_kernel(const int16_t *vol, int nx, int ny, int nz,
                                                               const double *pts, long long n, int cubic,
                                                               int gradient, double sx, double sy, double sz,
                                                               double *out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Block<LinearVol> b;
    b.vol.p = vol;
    b.vol.py = nx;
    b.vol.pz = (long long)nx * ny;
    b.ox = b.oy = b.oz = 0;
    b.ex = nx;
    b.ey = ny;
    b.ez = nz;
    double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    bool c = cubic != 0;
    if (!gradient) {
        out[i] = sample(b, x, y, z, c);
        return;
    }
    const double h = 0.5;  // _kernels.py:153-166
    double gx = sample(b, x + h, y, z, c) - sample(b, x - h, y, z, c);
    double gy = sample(b, x, y + h, z, c) - sample(b, x, y - h, z, c);
    double gz = sample(b, x, y, z + h, c) - sample(b, x, y, z - h, c);
    out[3 * i] = gx / sx;
    out[3 * i + 1] = gy / sy;
    out[3 * i + 2] = gz / sz;
}

// ---------------------------------------------------------- K4 measure

__global__ void __launch_bounds__(kBlock) threshold_kernel(const int16_t *__restrict__ v, long long n, int thr,
                                                           unsigned long long *count) {
#ifndef VR_K4_UNROLL
#define VR_K4_UNROLL 4
#endif
    constexpr int U = VR_K4_UNROLL;  // 16-byte loads in flight per thread (HBM latency x bandwidth)
    unsigned long long c = 0;
    const long long nvec = n / 8;
    const int4 *v8 = reinterpret_cast<const int4 *>(v);
    const long long stride = (long long)gridDim.x * blockDim.x;
    // each warp streams U consecutive 512-byte blocks per iteration (a
    // contiguous 2 KiB per warp, not U blocks a grid stride apart: DRAM
    // pages stay open -- 0.77 -> 0.86 of HBM at 512^3)
    const long long wstride = stride * U, lane = threadIdx.x & 31;
    const long long w0 = ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5) * (32 * U) + lane;
    const long long ustep = 32;
    for (long long i0 = w0; i0 < nvec; i0 += wstride) {
        int4 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) q[u] = i0 + u * ustep < nvec ? __ldcs(v8 + i0 + u * ustep) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (i0 + u * ustep >= nvec) continue;
            const int16_t *h = reinterpret_cast<const int16_t *>(&q[u]);
#pragma unroll
            for (int k = 0; k < 8; ++k) c += (h[k] >= thr) ? 1 : 0;
        }
    }
    for (long long i = nvec * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        c += (v[i] >= thr) ? 1 : 0;
    c = warp_sum(c);
    __shared__ unsigned long long part[kBlock / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < kBlock / 32; ++w) s += part[w];
        if (s) atomicAdd(count, s);
    }
}

// K0: one thread per sample, grid-stride (HBM-bound, runs once per volume)
template <typename T>
__global__ void __launch_bounds__(kBlock) ingest_kernel(const T *__restrict__ src, long long nxy, long long n,
                                                        const double *__restrict__ calib, int16_t *__restrict__ out,
                                                        unsigned long long *clamped) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int v = (int)__ldg(src + i);
        int16_t r;
        if (calib) {
            const long long z = i / nxy;
            const double cal = __ldg(calib + 2 * z) * (double)v + __ldg(calib + 2 * z + 1);
            c += (cal < -32768.0 || cal > 32767.0) ? 1 : 0;
            r = (int16_t)rint(cal < -32768.0 ? -32768.0 : (cal > 32767.0 ? 32767.0 : cal));
        } else {
            c += v > 32767 ? 1 : 0;  // u16 only; u8 / i16 never exceed (i32 is always calibrated)
            r = (int16_t)(v > 32767 ? 32767 : v);
        }
        out[i] = r;
    }
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(clamped, c);
}

}  // namespace

cudaError_t launch_value_range(const int16_t *vol, long long n, int *out, cudaStream_t s) {
    init_minmax_kernel<<<1, 32, 0, s>>>(out, 1);
    value_range_kernel<<<grid_for(n / 8 + 1, kBlock), kBlock, 0, s>>>(vol, n, out);
    return cudaGetLastError();
}

cudaError_t launch_phantom(int kind, int nx, int ny, int nz, int16_t *out, cudaStream_t s) {
    PhantomArgs p = {};
    p.kind = kind;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    if (kind == 2) {
        // phantoms.py:63-79: c(f) = f * n, s(f) = f * n in float64
        const double C[4][3] = {{0.50, 0.63, 0.63}, {0.50, 0.63, 0.71}, {0.34, 0.60, 0.55}, {0.68, 0.66, 0.56}};
        const double S[4][3] = {{0.46, 0.29, 0.29}, {0.40, 0.065, 0.065}, {0.17, 0.10, 0.08}, {0.12, 0.11, 0.09}};
        const double W[4] = {2.0, 1.5, 1.5, 1.5};
        for (int k = 0; k < 4; ++k) {
            Ellipsoid &e = p.e[k];
            e.cx = C[k][0] * nx;
            e.cy = C[k][1] * ny;
            e.cz = C[k][2] * nz;
            e.ax = S[k][0] * nx;
            e.ay = S[k][1] * ny;
            e.az = S[k][2] * nz;
            double m = e.ax;  // min(ax, ay, az)
            if (e.ay < m) m = e.ay;
            if (e.az < m) m = e.az;
            e.s_min = m;
            e.width = W[k];
        }
    } else if (kind == 0) {
        p.c[0] = nx / 2;
        p.c[1] = ny / 2;
        p.c[2] = nz / 2;
        int m = nx < ny ? nx : ny;
        m = m < nz ? m : nz;
        p.radius = (double)(m / 2);
    } else {
        p.c[0] = (nx - 1) / 2.0;
        p.c[1] = (ny - 1) / 2.0;
        p.c[2] = (nz - 1) / 2.0;
        int m = nx < ny ? nx : ny;
        m = m < nz ? m : nz;
        p.radius = m / 2.0;
        p.r_in = 0.55 * p.radius;
        p.r_out = 0.80 * p.radius;
    }
    long long n = (long long)nx * ny * nz;
    phantom_kernel<<<grid_for(n, kBlock, 64), kBlock, 0, s>>>(p, out);
    return cudaGetLastError();
}

static int zsplit_for(const Layout &L) {
    // one z-slice of a block per CTA (blocks skipped by the kernel exit at once)
    int bz = L.bsize < L.n[2] ? L.bsize : L.n[2];
    return bz < 1 ? 1 : (bz > 65535 ? 65535 : bz);
}

cudaError_t launch_block_minmax(const int16_t *vol, const Layout &L, int *vmin, int *vmax, cudaStream_t s) {
    int nblocks = L.nb[0] * L.nb[1] * L.nb[2];
    init_block_minmax_kernel<<<(nblocks + 255) / 256, 256, 0, s>>>(vmin, vmax, nblocks);
    dim3 grid(nblocks, zsplit_for(L));
    block_minmax_kernel<<<grid, kBlock, 0, s>>>(vol, L, vmin, vmax);
    return cudaGetLastError();
}

cudaError_t launch_visibility(const int16_t *bricks, const Layout &L, const VisArgs &v, cudaStream_t s) {
    size_t smem = (size_t)(v.nbins + 1) * sizeof(int);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(vis_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = launch_pdl(visbits_kernel, 2048 * 32 / kBlock, kBlock, 0, s, v);
    if (e != cudaSuccess) return e;
    e = launch_pdl(vis_setup_kernel, 1, kSetupThreads, smem, s, v);
    if (e != cudaSuccess) return e;
#ifndef VR_AABB_CTAS
#define VR_AABB_CTAS 8  // CTAs per SM (swept 2..16)
#endif
    e = launch_pdl(aabb_kernel, device_sms() * VR_AABB_CTAS, kAabbThreads, 0, s, bricks, L, v, zsplit_for(L));
    if (e != cudaSuccess) return e;
    e = launch_pdl(box_kernel, (v.nblocks + 127) / 128, 128, 0, s, L, v);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_brick_volume(const int16_t *vol, int nx, int ny, int nz, int16_t *bricks, cudaStream_t s) {
    int bnx = (nx + 3) / 4, bny = (ny + 3) / 4, bnz = (nz + 3) / 4;
    long long total = (long long)bnx * bny * bnz * 64;
    brick_kernel<<<grid_for(total, kBlock, 64), kBlock, 0, s>>>(vol, nx, ny, nz, bnx, bny, total, bricks);
    return cudaGetLastError();
}

// mcells[m] = union of the cells of the 16^3 macro cell m (4^3 cells)
__global__ void __launch_bounds__(kBlock) macro_from_cells_kernel(const short2 *__restrict__ cells, int ncx, int ncy,
                                                                  int ncz, int nmx, int nmy, int nmz, short2 *mcells) {
    const long long n = (long long)nmx * nmy * nmz;
    for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < n; m += (long long)gridDim.x * blockDim.x) {
        const int mx = (int)(m % nmx);
        const long long r = m / nmx;
        const int my = (int)(r % nmy), mz = (int)(r / nmy);
        int lo = INT_MAX, hi = INT_MIN;
        for (int i = 0; i < 64; ++i) {
            const int x = mx * 4 + (i & 3), y = my * 4 + ((i >> 2) & 3), z = mz * 4 + (i >> 4);
            if (x >= ncx || y >= ncy || z >= ncz) continue;
            const short2 b = __ldg(cells + ((long long)z * ncy + y) * ncx + x);
            lo = min(lo, (int)b.x);
            hi = max(hi, (int)b.y);
        }
        mcells[m] = make_short2((short)lo, (short)hi);
    }
}

// Raw footprint bounds for the pre-classified mode: rcells[c] = min / max of
// the voxels a sample based in cell c can read -- [4c-1, 4c+5] per axis (a
// Catmull-Rom base voxel g in [4c, 4c+3] reads g-1 .. g+2; block-local
// clamping only pulls taps inwards), clipped to the volume.  A cell whose raw
// voxels all classify to a zero alpha plane interpolates alpha exactly 0.
__global__ void __launch_bounds__(kBlock) raw_cell_kernel(const int16_t *__restrict__ vol, int nx, int ny, int nz,
                                                          int ncx, int ncy, int ncz, short2 *rcells) {
    const long long n = (long long)ncx * ncy * ncz;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
        const int cx = (int)(c % ncx);
        const long long r = c / ncx;
        const int cy = (int)(r % ncy), cz = (int)(r / ncy);
        const int x0 = max(4 * cx - 1, 0), x1 = min(4 * cx + 5, nx - 1);
        const int y0 = max(4 * cy - 1, 0), y1 = min(4 * cy + 5, ny - 1);
        const int z0 = max(4 * cz - 1, 0), z1 = min(4 * cz + 5, nz - 1);
        int lo = INT_MAX, hi = INT_MIN;
        for (int z = z0; z <= z1; ++z)
            for (int y = y0; y <= y1; ++y) {
                const int16_t *row = vol + ((long long)z * ny + y) * nx;
                for (int x = x0; x <= x1; ++x) {
                    const int v = __ldg(row + x);
                    lo = min(lo, v);
                    hi = max(hi, v);
                }
            }
        rcells[c] = make_short2((short)lo, (short)hi);
    }
}

cudaError_t launch_raw_bounds(const int16_t *vol, int nx, int ny, int nz, int ncx, int ncy, int ncz, short2 *rcells,
                              int nmx, int nmy, int nmz, short2 *rmcells, cudaStream_t s) {
    const long long nc = (long long)ncx * ncy * ncz;
    raw_cell_kernel<<<grid_for(nc, kBlock, 32), kBlock, 0, s>>>(vol, nx, ny, nz, ncx, ncy, ncz, rcells);
    const long long nm = (long long)nmx * nmy * nmz;
    macro_from_cells_kernel<<<grid_for(nm, kBlock, 32), kBlock, 0, s>>>(rcells, ncx, ncy, ncz, nmx, nmy, nmz,
                                                                             rmcells);
    return cudaGetLastError();
}

// Per frame, pre-classified mode: the smallest and largest int16 value in
// [vmin, vmax] whose pre-classified alpha plane is non-zero, i.e.
// rint(lut[classified_bin(v)].alpha * 255) >= 1 (as preclassify_kernel paints
// it); out = (INT_MAX, INT_MIN) when none.
__global__ void pre_range_kernel(const double *lut, int nbins, double lo, double bw, int vmin, int vmax, int *out) {
    pdl_enter();
    __shared__ int first, last;
    if (threadIdx.x == 0) {
        first = INT_MAX;
        last = INT_MIN;
    }
    __syncthreads();
    for (int v = vmin + (int)threadIdx.x; v <= vmax; v += blockDim.x) {
        const int k = classified_bin((double)v, lo, bw, nbins);
        if ((uint8_t)rint(__ldg(lut + 4 * k + 3) * 255.0) != 0) {
            atomicMin(&first, v);
            atomicMax(&last, v);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = first;
        out[1] = last;
    }
}

cudaError_t launch_pre_range(const double *lut, int nbins, double lut_lo, double bin_width, int vmin, int vmax,
                             int *out, cudaStream_t s) {
    cudaError_t e = launch_pdl(pre_range_kernel, 1, 1024, 0, s, lut, nbins, lut_lo, bin_width, vmin, vmax, out);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_interp_bounds(const int16_t *vol, int nx, int ny, int nz, int bnx, int bny, short2 *cubes,
                                 int ncx, int ncy, int ncz, short2 *cells, int nmx, int nmy, int nmz, short2 *mcells,
                                 cudaStream_t s) {
    dim3 grid((nx + kCubeTile - 1) / kCubeTile, (ny + kCubeTile - 1) / kCubeTile, (nz + kCubeTile - 1) / kCubeTile);
    cube_bound_kernel<<<grid, 512, 0, s>>>(vol, nx, ny, nz, bnx, bny, cubes);
    const long long nc = (long long)ncx * ncy * ncz;
    cell_from_cubes_kernel<<<grid_for(nc, kBlock, 32), kBlock, 0, s>>>(cubes, nx, ny, nz, ncx, ncy, ncz, cells);
    const long long nm = (long long)nmx * nmy * nmz;
    macro_from_cells_kernel<<<grid_for(nm, kBlock, 32), kBlock, 0, s>>>(cells, ncx, ncy, ncz, nmx, nmy, nmz,
                                                                             mcells);
    return cudaGetLastError();
}

cudaError_t launch_lut_range(const double *lut, int nbins, double lut_lo, double lut_inv_w, int *range,
                             const ZeroSpec &zero, cudaStream_t s) {
    cudaError_t e = launch_pdl(lut_range_kernel, 1, kSetupThreads, 0, s, lut, nbins, lut_lo, lut_inv_w, range, zero);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_tbl_nonzero(const double *table, int n, int *nz, cudaStream_t s) {
    cudaError_t e = launch_pdl(tbl_nonzero_kernel, 1, 1024, 0, s, table, n, nz);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// x-quad texture for the sampling-path A/B (VR_SAMPLER_TEX builds)
__global__ void xquad_kernel(const int16_t *__restrict__ v, int nx, int ny, int nz, cudaSurfaceObject_t surf) {
    const long long n = (long long)nx * ny * nz;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % nx);
        const long long r = i / nx;
        const int y = (int)(r % ny), z = (int)(r / ny);
        const int16_t *row = v + r * nx;
        const short4 q = make_short4(row[x], row[min(x + 1, nx - 1)], row[min(x + 2, nx - 1)], row[min(x + 3, nx - 1)]);
        surf3Dwrite(q, surf, x * (int)sizeof(short4), y, z);
    }
}

cudaError_t launch_xquads(const int16_t *vol, int nx, int ny, int nz, unsigned long long surf, cudaStream_t s) {
    xquad_kernel<<<grid_for((long long)nx * ny * nz, kBlock, 16), kBlock, 0, s>>>(vol, nx, ny, nz,
                                                                                (cudaSurfaceObject_t)surf);
    return cudaGetLastError();
}

cudaError_t launch_count_hits(const uint8_t *hits, int n, int nviews, unsigned long long *totals,
                              const unsigned long long *vis_counters, cudaStream_t s) {
    cudaError_t e = launch_pdl(count_hits_kernel, nviews, 1024, 0, s, hits, n, totals, vis_counters);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_preclassify(const int16_t *vol, long long n, const double *lut, int nbins, double lut_lo,
                               double bin_width, uint8_t *rgba, cudaStream_t s) {
    preclassify_kernel<<<grid_for(n, kBlock, 64), kBlock, 0, s>>>(vol, n, lut, nbins, lut_lo, bin_width, rgba);
    return cudaGetLastError();
}

cudaError_t launch_sample_points(const int16_t *vol, int nx, int ny, int nz, const double *pts, long long n,
                                 int cubic, int gradient, double sx, double sy, double sz, double *out,
                                 cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    long long g = (n + kBlock - 1) / kBlock;
    sample_points_kernel<<<(unsigned)g, kBlock, 0, s>>>(vol, nx, ny, nz, pts, n, cubic, gradient, sx, sy, sz, out);
    return cudaGetLastError();
}

cudaError_t launch_threshold_count(const int16_t *vol, long long n, int thr, unsigned long long *count,
                                   cudaStream_t s) {
    threshold_kernel<<<grid_for(n / 8 + 1, kBlock, 8), kBlock, 0, s>>>(vol, n, thr, count);
    return cudaGetLastError();
}

cudaError_t launch_ingest(const void *src, int format, long long nxy, int nz, const double *calib,
                          int16_t *out, unsigned long long *clamped, cudaStream_t s) {
    const long long n = nxy * nz;
    const int grid = grid_for(n, kBlock, 16);
    if (format == kFormatU8)
        ingest_kernel<<<grid, kBlock, 0, s>>>(static_cast<const uint8_t *>(src), nxy, n, calib, out, clamped);
    else if (format == kFormatI16)
        ingest_kernel<<<grid, kBlock, 0, s>>>(static_cast<const int16_t *>(src), nxy, n, calib, out, clamped);
    else if (format == kFormatU16)
        ingest_kernel<<<grid, kBlock, 0, s>>>(static_cast<const uint16_t *>(src), nxy, n, calib, out, clamped);
    else
        ingest_kernel<<<grid, kBlock, 0, s>>>(static_cast<const int32_t *>(src), nxy, n, calib, out, clamped);
    return cudaGetLastError();
}


}  // namespace vr
