// vr_measure.cu -- K4: the paper's "method of spheres" on
// the voxel grid.  The reference measures S (surface area inside a probe ball)
// and V (object volume inside it) on triangle meshes by Monte Carlo
// (/root/reference/pkg/src/voxelray/morphology.py:70-143 clipped_area,
// :238-267 clipped_volume, :270-306 svr_at_point); it has no voxel form
// (SURVEY G2).  Here, on the CT volume itself, exactly:
//
//  * V: voxels with value >= thr (centre inside the closed ball for the ball
//    form) -- an integer count, V = count * sx*sy*sz;
//  * S: area of the isosurface at level L = thr - 0.5 of the piecewise-linear
//    (Kuhn-tetrahedra) interpolant -- for integer voxels v >= thr <=> v > L, so
//    the surface separates exactly the voxels V counts.  Cells are the unit
//    cubes between voxel centres, padded by one cell on every side with the
//    outside value -32768 (the surface closes at the volume border); each cell
//    splits into the 6 tetrahedra 000 -> e_a -> e_a+e_b -> 111, in each of
//    which the level set is a triangle or a planar quad.  Every polygon's area
//    is rounded to a multiple of 2^-24 mm^2 and summed in 64-bit integers, so
//    the sum is independent of summation order and bit-exact against the C
//    restatement (oracle/vr_oracle.c vro_threshold_measure / vro_ball_measure:
//    same float64 operations, same order, no FMA).  The ball form keeps the
//    polygons whose vertex centroid lies in the closed ball.
//
// Parity of the definition cannot be pinned to a reference function (there is
// none); tests/test_measure.py pins it to the analytic oracles of
// SPEC.md:472-473 (flat face SVR -> 3/(2R), enclosed sphere SVR -> 3/a).
//
// The whole-volume measure is three passes: (1) the only pass over the int16
// voxels -- every voxel's inside bit into a flat bit array (1/16 of the
// volume, L2-resident) and the count V, HBM-bound; (2a) a scan of the bit
// array for cells whose eight corners disagree, appended to a list; (2b) the
// tetrahedra for the listed cells, one per thread.  The ball form scans the
// bit array inside each ball's bounding box.
#include <cstdint>

#include "vr_common.cuh"
#include "vr_prep.cuh"

namespace vr {
namespace {

constexpr int kMeasureThreads = 256;
constexpr double kAreaScale = 16777216.0;  // 2^24
constexpr int kBallSplit = 8;  // CTAs per probe ball

// Cell corner c (bit 0: x, 1: y, 2: z) of the cell with base voxel (cx, cy,
// cz), in mm (voxel centres at index * spacing).
struct CellGeom {
    int cx, cy, cz;
    double sx, sy, sz;
    VR_D double px(int c) const { return (double)(cx + (c & 1)) * sx; }
    VR_D double py(int c) const { return (double)(cy + ((c >> 1) & 1)) * sy; }
    VR_D double pz(int c) const { return (double)(cz + ((c >> 2) & 1)) * sz; }
};

// the level-set point on edge (p inside, q outside): t = f_p / (f_p - f_q) from p
VR_D void edge_point(const CellGeom &G, int p, int q, double fp, double fq, double *out) {
    const double t = fp / (fp - fq);
    const double Px = G.px(p), Py = G.py(p), Pz = G.pz(p);
    out[0] = Px + t * (G.px(q) - Px);
    out[1] = Py + t * (G.py(q) - Py);
    out[2] = Pz + t * (G.pz(q) - Pz);
}

VR_D double cross_half_norm(double ux, double uy, double uz, double wx, double wy, double wz) {
    const double cx = uy * wz - uz * wy;
    const double cy = uz * wx - ux * wz;
    const double cz = ux * wy - uy * wx;
    return 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
}

// Fixed-point area of one cell's level-set polygons (corner c = x | y<<1 | z<<2
// with field f[c] = v - L); BALL keeps only polygons whose centroid lies in
// the closed ball (bx, by, bz, r2).
template <bool BALL>
VR_D unsigned long long cell_area_fx(const double f[8], const CellGeom &G, double bx, double by, double bz, double r2) {
    unsigned long long acc = 0;
    unsigned inside = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) inside |= (f[c] > 0.0 ? 1u : 0u) << c;
#pragma unroll 1
    for (int t = 0; t < 6; ++t) {
        // Kuhn permutations (0,1,2),(0,2,1),(1,0,2),(1,2,0),(2,0,1),(2,1,0)
        const int p0 = t >> 1;
        const int p1 = (t == 0 || t == 5) ? 1 : ((t == 1 || t == 3) ? 2 : 0);
        const int v1 = 1 << p0, v2 = v1 | (1 << p1);
        const int v[4] = {0, v1, v2, 7};
        int in[4], out[4], ni = 0, no = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if ((inside >> v[c]) & 1u)
                in[ni++] = v[c];
            else
                out[no++] = v[c];
        }
        if (ni == 0 || no == 0) continue;
        double a[3], b[3], c3[3], d[3], area, gx, gy, gz;
        if (ni == 1 || no == 1) {
            if (ni == 1) {
                edge_point(G, in[0], out[0], f[in[0]], f[out[0]], a);
                edge_point(G, in[0], out[1], f[in[0]], f[out[1]], b);
                edge_point(G, in[0], out[2], f[in[0]], f[out[2]], c3);
            } else {
                edge_point(G, in[0], out[0], f[in[0]], f[out[0]], a);
                edge_point(G, in[1], out[0], f[in[1]], f[out[0]], b);
                edge_point(G, in[2], out[0], f[in[2]], f[out[0]], c3);
            }
            area = cross_half_norm(b[0] - a[0], b[1] - a[1], b[2] - a[2], c3[0] - a[0], c3[1] - a[1], c3[2] - a[2]);
            if (BALL) {
                gx = ((a[0] + b[0]) + c3[0]) / 3.0;
                gy = ((a[1] + b[1]) + c3[1]) / 3.0;
                gz = ((a[2] + b[2]) + c3[2]) / 3.0;
            }
        } else {
            // planar quad (in0,out0) (in0,out1) (in1,out1) (in1,out0)
            edge_point(G, in[0], out[0], f[in[0]], f[out[0]], a);
            edge_point(G, in[0], out[1], f[in[0]], f[out[1]], b);
            edge_point(G, in[1], out[1], f[in[1]], f[out[1]], c3);
            edge_point(G, in[1], out[0], f[in[1]], f[out[0]], d);
            area = cross_half_norm(c3[0] - a[0], c3[1] - a[1], c3[2] - a[2], d[0] - b[0], d[1] - b[1], d[2] - b[2]);
            if (BALL) {
                gx = (((a[0] + b[0]) + c3[0]) + d[0]) * 0.25;
                gy = (((a[1] + b[1]) + c3[1]) + d[1]) * 0.25;
                gz = (((a[2] + b[2]) + c3[2]) + d[2]) * 0.25;
            }
        }
        if (BALL) {
            const double dx = gx - bx, dy = gy - by, dz = gz - bz;
            if (!((dx * dx + dy * dy) + dz * dz <= r2)) continue;
        }
        acc += (unsigned long long)llrint(area * kAreaScale);
    }
    return acc;
}

VR_D unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One CTA-wide sum of (count, area) into out[0..1].
VR_D void cta_accumulate(unsigned long long c, unsigned long long area, unsigned long long *out_c,
                         unsigned long long *out_a, bool store) {
    __shared__ unsigned long long part[2][kMeasureThreads / 32];
    c = warp_sum64(c);
    area = warp_sum64(area);
    if ((threadIdx.x & 31) == 0) {
        part[0][threadIdx.x >> 5] = c;
        part[1][threadIdx.x >> 5] = area;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        unsigned long long s = 0;
        for (int w = 0; w < kMeasureThreads / 32; ++w) s += part[threadIdx.x][w];
        unsigned long long *dst = threadIdx.x == 0 ? out_c : out_a;
        if (dst) {
            if (store)
                *dst = s;
            else if (s)
                atomicAdd(dst, s);
        }
    }
}

struct MeasureVol {
    const int16_t *v;
    int nx, ny, nz;
    double sx, sy, sz;
};

VR_D int voxel_or_pad(const MeasureVol &m, int i, int j, int k) {
    if (i < 0 || j < 0 || k < 0 || i >= m.nx || j >= m.ny || k >= m.nz) return -32768;
    return __ldg(m.v + ((long long)k * m.ny + j) * m.nx + i);
}

// first / last cell index of a ball's bounding box, clamped to [-1, n-1] in
// floating point first (no overflow for balls far outside the volume)
VR_D int box_lo(double lo_mm, double s) {
    const double v = floor(lo_mm / s) - 1.0;
    return v < -1.0 ? -1 : (v > 2.0e9 ? 2000000000 : (int)v);
}
VR_D int box_hi(double hi_mm, double s, int n) {
    const double v = ceil(hi_mm / s) + 1.0;
    return v > (double)(n - 1) ? n - 1 : (v < -2.0e9 ? -2000000000 : (int)v);
}

// ------------------------------------------------ two-pass fast path
// Pass 1 (HBM-bound, the only pass over the int16 voxels): every voxel's
// inside bit (v >= thr) into a flat bit array -- bit i of word i/32 is voxel
// i in (z, y, x) order, 1/16 of the volume (16 MiB at 512^3, L2-resident) --
// and the voxel count V.  A lane reads 16 bytes (8 voxels), four lanes merge
// their bytes into one 32-bit word: every load and store is coalesced.
// Pass 2 (L2-bound): per cell row (cy, cz) and 32-cell chunk, the 33-bit
// windows of its four voxel rows locate the cells whose corners are not all
// equal; only those (a few per mille at CT thresholds) read their 8 voxels
// and run the tetrahedra.
// 8 inside bits (v >= thr) of the 8 voxels of a 16-byte group
#ifndef VR_K4_SIMD
#define VR_K4_SIMD 1  // whole-volume measure 155 -> 147 us, balls 268 -> 260 us
#endif
VR_D unsigned group_bits(const int4 q, int thr) {
#if VR_K4_SIMD
    // two 16-bit compares per instruction; thr outside int16 is all or none
    if (thr <= -32768) return 0xffu;
    if (thr > 32767) return 0u;
    const unsigned t2 = ((unsigned)thr & 0xffffu) * 0x10001u;
    const unsigned m0 = __vcmpges2((unsigned)q.x, t2), m1 = __vcmpges2((unsigned)q.y, t2);
    const unsigned m2 = __vcmpges2((unsigned)q.z, t2), m3 = __vcmpges2((unsigned)q.w, t2);
    // low halves -> bits 0, 2, 4, 6 and high halves -> bits 16, 18, 20, 22
    const unsigned b = (m0 & 0x10001u) | ((m1 & 0x10001u) << 2) | ((m2 & 0x10001u) << 4) | ((m3 & 0x10001u) << 6);
    return (b & 0xffu) | ((b >> 15) & 0xffu);
#else
    const unsigned w[4] = {(unsigned)q.x, (unsigned)q.y, (unsigned)q.z, (unsigned)q.w};
    unsigned b = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        b |= ((int)(short)(w[k] & 0xffffu) >= thr ? 1u : 0u) << (2 * k);
        b |= ((int)(short)(w[k] >> 16) >= thr ? 1u : 0u) << (2 * k + 1);
    }
    return b;
#endif
}

#ifndef VR_K4_UNROLL
#define VR_K4_UNROLL 4
#endif
constexpr int kBitsUnroll = VR_K4_UNROLL;  // 16-byte loads in flight per lane (HBM latency x bandwidth)

__global__ void __launch_bounds__(kMeasureThreads) inside_bits_kernel(const int16_t *__restrict__ v, long long n,
                                                                      int thr, unsigned *__restrict__ bits,
                                                                      unsigned long long *count) {
    const long long n8 = n >> 3;  // whole 8-voxel groups
    const int lane = threadIdx.x & 31;
    unsigned long long c = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int4 *v4 = reinterpret_cast<const int4 *>(v);
    const long long tail_word = (n & 31) ? (n >> 5) : -1;  // owned by the tail thread
    // warp-uniform trip counts (whole warps of groups): the shuffles below run
    // converged; kBitsUnroll independent loads are issued before any is used
    // each warp streams kBitsUnroll consecutive 512-byte blocks per
    // iteration (contiguous, so DRAM pages stay open)
    const long long gbase = ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5) * (32 * kBitsUnroll);
    const long long ustep = 32;
    for (long long g0 = gbase; g0 < n8; g0 += kBitsUnroll * stride) {
        int4 q[kBitsUnroll];
#pragma unroll
        for (int u = 0; u < kBitsUnroll; ++u) {
            const long long g = g0 + u * ustep + lane;
            q[u] = g < n8 ? __ldcs(v4 + g) : make_int4(0, 0, 0, 0);  // streamed: read once
        }
#pragma unroll
        for (int u = 0; u < kBitsUnroll; ++u) {
            const long long g = g0 + u * ustep + lane;
            const unsigned b = g < n8 ? group_bits(q[u], thr) : 0u;
            c += (unsigned long long)__popc(b);
            // lanes 4m .. 4m+3 hold voxels 32m' .. 32m'+31 of one word
            unsigned word = b << (8 * (lane & 3));
            word |= __shfl_xor_sync(0xffffffffu, word, 1);
            word |= __shfl_xor_sync(0xffffffffu, word, 2);
            if ((lane & 3) == 0 && g < n8 && (g >> 2) != tail_word) bits[g >> 2] = word;
        }
    }
    // tail voxels (n % 8) and the tail word's missing lanes: one thread
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 31)) {
        const long long w0 = n >> 5;
        unsigned word = 0;
        for (long long i = w0 << 5; i < n; ++i) {
            const bool in = v[i] >= thr;
            word |= (in ? 1u : 0u) << (i & 31);
            if (i >= (n8 << 3)) c += in ? 1 : 0;
        }
        bits[w0] = word;
    }
    const unsigned long long cs = warp_sum64(c);
    if (lane == 0 && cs) atomicAdd(count, cs);
}

// bits of voxels x0 .. x0+32 of row (j, k) (bit b = voxel x0+b; outside the
// volume: 0), from the flat bit array
VR_D unsigned long long row_bits33(const MeasureVol &m, const unsigned *bits, int x0, int j, int k) {
    if (j < 0 || k < 0 || j >= m.ny || k >= m.nz) return 0ull;
    const int lo = x0 < 0 ? 0 : x0;
    const int hi = x0 + 32 < m.nx - 1 ? x0 + 32 : m.nx - 1;  // last voxel wanted
    if (lo > hi) return 0ull;
    const long long b0 = ((long long)k * m.ny + j) * m.nx + lo;
    const long long w = b0 >> 5;
    const int sh = (int)(b0 & 31);
    // (the bit array has a spare word after the last one: reading w + 1 is safe)
    const unsigned long long win = (unsigned long long)__ldg(bits + w) | ((unsigned long long)__ldg(bits + w + 1) << 32);
    unsigned long long r = win >> sh;  // >= 33 valid bits (sh <= 31)
    const int len = hi - lo + 1;
    r &= len >= 64 ? ~0ull : ((1ull << len) - 1ull);
    return r << (lo - x0);
}

// position of the k-th (0-based) set bit of m
VR_D int nth_set_bit(unsigned m, int k) {
    int pos = 0;
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const int c = __popc(m & ((1u << w) - 1u));
        if (k >= c) {
            k -= c;
            m >>= w;
            pos += w;
        }
    }
    return pos;
}

// The straddling cells of all 32 lanes (lane l: cells x0_l + b for the set
// bits b of st_l, row (cy_l, cz_l)) spread evenly over the lanes -- 32 cells
// per round -- so the tetrahedra run at full SIMT width however unevenly the
// surface crosses the lanes' chunks.  Every lane of the warp must call this;
// returns this lane's share of the fixed-point area.
template <bool BALL>
VR_D unsigned long long warp_cells_area(const MeasureVol &m, unsigned st, int x0, int cy, int cz, double level,
                                        double bx, double by, double bz, double r2) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int cnt = __popc(st);
    int incl = cnt;  // inclusive prefix of the counts over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(full, incl, 31);
    const int base = incl - cnt;
    unsigned long long area = 0;
    for (int start = 0; start < total; start += 32) {
        const int id = start + lane;
        int src = 0;  // the last lane whose base <= id
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const int cand = src + step;
            const int b = __shfl_sync(full, base, cand & 31);
            if (cand < 32 && b <= id) src = cand;
        }
        const int k = id - __shfl_sync(full, base, src);
        const unsigned ms = __shfl_sync(full, st, src);
        const int sx0 = __shfl_sync(full, x0, src), scy = __shfl_sync(full, cy, src), scz = __shfl_sync(full, cz, src);
        if (id < total) {
            const int cx = sx0 + nth_set_bit(ms, k);
            double f[8];
#pragma unroll
            for (int c = 0; c < 8; ++c)
                f[c] = (double)voxel_or_pad(m, cx + (c & 1), scy + ((c >> 1) & 1), scz + ((c >> 2) & 1)) - level;
            const CellGeom G{cx, scy, scz, m.sx, m.sy, m.sz};
            area += cell_area_fx<BALL>(f, G, bx, by, bz, r2);
        }
    }
    return area;
}

// cells x0 .. x0+31 of cell row (cy, cz) whose 8 corner bits are not all equal
VR_D unsigned long long chunk_straddle(const MeasureVol &m, const unsigned *bits, int x0, int cy, int cz) {
    const unsigned long long r0 = row_bits33(m, bits, x0, cy, cz), r1 = row_bits33(m, bits, x0, cy + 1, cz);
    const unsigned long long r2 = row_bits33(m, bits, x0, cy, cz + 1), r3 = row_bits33(m, bits, x0, cy + 1, cz + 1);
    const unsigned long long all = r0 & r1 & r2 & r3, any = r0 | r1 | r2 | r3;
    unsigned long long st = ((any | (any >> 1)) & ~(all & (all >> 1))) & 0xffffffffull;
    const int ncells = m.nx - x0;  // cells x0 .. nx-1 exist (cx <= nx-1)
    if (ncells < 32) st &= ncells <= 0 ? 0ull : ((1ull << ncells) - 1ull);
    return st;
}

// Pass 2a, whole volume: the straddling cells of every (32-cell chunk, cell
// row, cell slab), appended to a list (one warp-aggregated atomic per warp);
// a lean kernel (no float64), so it runs at full occupancy over the L2-
// resident bit array.  Cells are packed as (cx + 1) | (cy + 1) << 21 |
// (cz + 1) << 42.  Returns the list length in *ncells (capped at cap; the
// overflow count is what tells the host to fall back, see the launcher).
#ifndef VR_SCAN_SLABS
#define VR_SCAN_SLABS 4  // measured at 512^3: 2: 160 us, 4: 156, 8: 158, 16: 173, 32: 190 (whole measure)
#endif
constexpr int kScanSlabs = VR_SCAN_SLABS;  // cell slabs per thread of the straddle scan (the z window slides)

__global__ void __launch_bounds__(kMeasureThreads) straddle_scan_kernel(MeasureVol m, const unsigned *__restrict__ bits,
                                                                        int nchunks, unsigned long long *list,
                                                                        unsigned long long cap,
                                                                        unsigned long long *ncells) {
    // thread = (32-cell chunk, cell row, run of kScanSlabs cell slabs): the
    // upper voxel rows of one slab are the lower rows of the next, so each
    // step fetches two rows instead of four.  (32-bit index arithmetic: the
    // launcher checks the counts.)
    const int nseg = (m.nz + 1 + kScanSlabs - 1) / kScanSlabs;
    const int total = nchunks * (m.ny + 1) * nseg;
    const int lane = threadIdx.x & 31;
    for (int t0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) & ~31u); t0 < total; t0 += gridDim.x * blockDim.x) {
        const int t = t0 + lane;
        const bool valid = t < total;
        const int tc = valid ? t : 0;
        const int c = tc % nchunks;
        const int r = tc / nchunks;
        const int cy = r % (m.ny + 1) - 1;
        const int cz0 = (r / (m.ny + 1)) * kScanSlabs - 1;
        const int x0 = 32 * c - 1;
        const int ncl = m.nx - x0;  // cells x0 .. nx-1 exist (cx <= nx-1)
        const unsigned long long cmask = ncl >= 32 ? 0xffffffffull : (ncl <= 0 ? 0ull : ((1ull << ncl) - 1ull));
        unsigned long long lo0 = row_bits33(m, bits, x0, cy, cz0), lo1 = row_bits33(m, bits, x0, cy + 1, cz0);
        const unsigned long long yz0 = ((unsigned long long)(cy + 1) << 21);
        for (int k = 0; k < kScanSlabs; ++k) {
            const int cz = cz0 + k;
            const bool live = valid && cz < m.nz;  // cell slabs -1 .. nz-1
            unsigned long long hi0 = 0, hi1 = 0;
            if (live) {
                hi0 = row_bits33(m, bits, x0, cy, cz + 1);
                hi1 = row_bits33(m, bits, x0, cy + 1, cz + 1);
            }
            const unsigned long long all = lo0 & lo1 & hi0 & hi1, any = lo0 | lo1 | hi0 | hi1;
            unsigned st = live ? (unsigned)(((any | (any >> 1)) & ~(all & (all >> 1))) & cmask) : 0u;
            lo0 = hi0;
            lo1 = hi1;
            if (!__any_sync(0xffffffffu, st != 0u)) continue;  // (most steps: no straddling cell)
            const int cnt = __popc(st);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int wtotal = __shfl_sync(0xffffffffu, incl, 31);
            unsigned long long base = 0;
            if (lane == 31) base = atomicAdd(ncells, (unsigned long long)wtotal);
            base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(incl - cnt);
            const unsigned long long yz = yz0 | ((unsigned long long)(cz + 1) << 42);
            while (st) {
                const int b = __ffs(st) - 1;
                st &= st - 1;
                if (base < cap) list[base] = (unsigned long long)(x0 + b + 1) | yz;
                ++base;
            }
        }
    }
}

// Pass 2b: one straddling cell per thread: its 8 voxels, the tetrahedra.
__global__ void __launch_bounds__(kMeasureThreads) cell_area_kernel(MeasureVol m, int thr,
                                                                    const unsigned long long *__restrict__ list,
                                                                    const unsigned long long *ncells,
                                                                    unsigned long long cap, unsigned long long *out) {
    const double level = (double)thr - 0.5;
    const unsigned long long n = *ncells <= cap ? *ncells : 0ull;  // overflow: surface_kernel instead
    unsigned long long area = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long e = __ldg(list + i);
        const int cx = (int)(e & 0x1fffff) - 1, cy = (int)((e >> 21) & 0x1fffff) - 1, cz = (int)(e >> 42) - 1;
        double f[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
            f[c] = (double)voxel_or_pad(m, cx + (c & 1), cy + ((c >> 1) & 1), cz + ((c >> 2) & 1)) - level;
        const CellGeom G{cx, cy, cz, m.sx, m.sy, m.sz};
        area += cell_area_fx<false>(f, G, 0.0, 0.0, 0.0, 0.0);
    }
    cta_accumulate(0, area, nullptr, out + 1, false);
}

// Pass 2 (fallback when the cell list overflows): thread = (32-cell chunk,
// cell row), the tetrahedra shared out warp-wide.
__global__ void __launch_bounds__(kMeasureThreads) surface_kernel(MeasureVol m, const unsigned *__restrict__ bits,
                                                                  int thr, int nchunks, const unsigned long long *ncells,
                                                                  unsigned long long cap, unsigned long long *out) {
    if (*ncells <= cap) return;  // the list held every straddling cell: cell_area_kernel did the work
    const double level = (double)thr - 0.5;
    unsigned long long area = 0;
    const long long total = (long long)nchunks * (m.ny + 1) * (m.nz + 1);
    for (long long t0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) & ~31ll; t0 < total;
         t0 += (long long)gridDim.x * blockDim.x) {
        const long long t = t0 + (threadIdx.x & 31);
        unsigned st = 0;
        int x0 = 0, cy = 0, cz = 0;
        if (t < total) {
            const int c = (int)(t % nchunks);
            const long long r = t / nchunks;
            cy = (int)(r % (m.ny + 1)) - 1;
            cz = (int)(r / (m.ny + 1)) - 1;
            x0 = 32 * c - 1;
            st = (unsigned)chunk_straddle(m, bits, x0, cy, cz);
        }
        if (__any_sync(0xffffffffu, st != 0u))
            area += warp_cells_area<false>(m, st, x0, cy, cz, level, 0.0, 0.0, 0.0, 0.0);
    }
    cta_accumulate(0, area, nullptr, out + 1, false);
}

// Pass 2 per ball: one CTA per ball; thread = (32-cell chunk, cell row, cell
// slab) of the ball's bounding box.  V: the inside voxels of row
// (cy, cz) whose centres lie in the ball; S: the straddling cells' polygons
// with centroid in the ball.
__global__ void __launch_bounds__(kMeasureThreads) ball_surface_kernel(MeasureVol m, const unsigned *__restrict__ bits,
                                                                       int thr, const double *centres,
                                                                       const double *radii, unsigned long long *counts,
                                                                       unsigned long long *areas) {
    const int ball = blockIdx.x;
    const double bx = centres[3 * ball], by = centres[3 * ball + 1], bz = centres[3 * ball + 2];
    const double rad = radii[ball];
    const double r2 = rad * rad;
    const double level = (double)thr - 0.5;
    const int i0 = box_lo(bx - rad, m.sx), i1 = box_hi(bx + rad, m.sx, m.nx);
    const int j0 = box_lo(by - rad, m.sy), j1 = box_hi(by + rad, m.sy, m.ny);
    const int k0 = box_lo(bz - rad, m.sz), k1 = box_hi(bz + rad, m.sz, m.nz);
    unsigned long long count = 0, area = 0;
    if (i0 <= i1 && j0 <= j1 && k0 <= k1) {
        const int nc = (i1 - i0) / 32 + 1, nj = j1 - j0 + 1;
        const int items = nc * nj * (k1 - k0 + 1);  // (32-cell chunk, cell row, cell slab)
        // warp-uniform trip counts: tetrahedra shared out warp-wide; the
        // ball's items are split over gridDim.y CTAs (counts added atomically)
        const int stride = (int)(blockDim.x * gridDim.y);
        for (int t0 = (int)(blockIdx.y * blockDim.x + (threadIdx.x & ~31u)); t0 < items; t0 += stride) {
            const int t = t0 + (threadIdx.x & 31);
            const bool valid = t < items;
            const int tc = valid ? t : 0;
            const int x0 = i0 + 32 * (tc % nc), cy = j0 + (tc / nc) % nj, cz = k0 + tc / (nc * nj);
            const int xe = min(x0 + 31, i1);  // this chunk's last cell
            const unsigned long long keep = valid ? (2ull << (xe - x0)) - 1ull : 0ull;
            const unsigned st = (unsigned)(valid ? chunk_straddle(m, bits, x0, cy, cz) & keep : 0ull);
            if (areas && __any_sync(0xffffffffu, st != 0u))
                area += warp_cells_area<true>(m, st, x0, cy, cz, level, bx, by, bz, r2);
            // voxels x0 .. xe of row (cy, cz) (cells at negative indices have no base voxel)
            unsigned long long in = valid ? row_bits33(m, bits, x0, cy, cz) & keep : 0ull;
            while (in) {
                const int b = __ffsll((long long)in) - 1;
                in &= in - 1;
                const double dx = (double)(x0 + b) * m.sx - bx, dy = (double)cy * m.sy - by;
                const double dz = (double)cz * m.sz - bz;
                count += ((dx * dx + dy * dy) + dz * dz <= r2) ? 1 : 0;
            }
        }
    }
    cta_accumulate(count, area, counts + ball, areas ? areas + ball : nullptr, false);
}

}  // namespace

// stream-ordered scratch for the inside-bit array (freed on the stream)
struct BitsScratch {
    cudaStream_t s;
    unsigned *p = nullptr;
    unsigned long long *count = nullptr;  // a spare counter after the bits
    explicit BitsScratch(cudaStream_t st) : s(st) {}
    cudaError_t alloc(long long nvox) {
        const size_t words = (size_t)((nvox + 31) / 32 + 1) & ~(size_t)1;  // even: the counter is 8-byte aligned
        cudaError_t e = cudaMallocAsync((void **)&p, words * 4 + 8, s);
        if (e == cudaSuccess) count = reinterpret_cast<unsigned long long *>(p + words);
        return e;
    }
    ~BitsScratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

cudaError_t launch_inside_bits(const int16_t *vol, long long n, int thr, unsigned *bits, unsigned long long *count,
                               cudaStream_t s) {
    long long grid = (n / 8 + kMeasureThreads - 1) / kMeasureThreads;
    const long long cap = (long long)device_sms() * 16;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    inside_bits_kernel<<<(unsigned)grid, kMeasureThreads, 0, s>>>(vol, n, thr, bits, count);
    return cudaGetLastError();
}

cudaError_t launch_threshold_measure(const int16_t *vol, int nx, int ny, int nz, double sx, double sy, double sz,
                                     int thr, unsigned long long *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    MeasureVol m{vol, nx, ny, nz, sx, sy, sz};
    const long long n = (long long)nx * ny * nz;
    // (volumes are cudaMalloc allocations: 256-byte aligned, as the 16-byte loads need)
    if ((reinterpret_cast<uintptr_t>(vol) & 15) != 0) return cudaErrorMisalignedAddress;
    BitsScratch bits(s);
    if ((e = bits.alloc(n)) != cudaSuccess) return e;
    if ((e = launch_inside_bits(vol, n, thr, bits.p, out, s)) != cudaSuccess) return e;
    const int nchunks = (nx + 1 + 31) / 32;  // cells -1 .. nx-1 in chunks of 32
    const long long total = (long long)nchunks * (ny + 1) * (nz + 1);
    if (total >= (1ll << 31)) return cudaErrorInvalidValue;  // > 2^36 voxels: not a CT volume
    long long grid = (total + kMeasureThreads - 1) / kMeasureThreads;
    const long long cap_ctas = (long long)device_sms() * 16;
    if (grid > cap_ctas) grid = cap_ctas;
    const long long scan_items = (long long)nchunks * (ny + 1) * ((nz + 1 + kScanSlabs - 1) / kScanSlabs);
    long long scan_grid = (scan_items + kMeasureThreads - 1) / kMeasureThreads;
    if (scan_grid > cap_ctas) scan_grid = cap_ctas;
    // straddling cells: the list holds up to 1/16 of all cells (every
    // boundary of a 512^3 CT at its bone threshold is ~0.2 %); beyond
    // that the one-pass surface kernel (correct for any count) runs
    // instead, chosen on the device so nothing waits on the host
    const unsigned long long cap = (unsigned long long)((long long)(nx + 1) * (ny + 1) * (nz + 1) / 16 + 1024);
    void *lst = nullptr;
    if ((e = cudaMallocAsync(&lst, (size_t)cap * 8 + 16, s)) != cudaSuccess) return e;
    unsigned long long *ncells = reinterpret_cast<unsigned long long *>((char *)lst + (size_t)cap * 8);
    e = cudaMemsetAsync(ncells, 0, 8, s);
    if (e == cudaSuccess) {
        straddle_scan_kernel<<<(unsigned)scan_grid, kMeasureThreads, 0, s>>>(m, bits.p, nchunks,
                                                                        (unsigned long long *)lst, cap, ncells);
        cell_area_kernel<<<(unsigned)device_sms() * 8, kMeasureThreads, 0, s>>>(
            m, thr, (const unsigned long long *)lst, ncells, cap, out);
        surface_kernel<<<(unsigned)grid, kMeasureThreads, 0, s>>>(m, bits.p, thr, nchunks, ncells, cap, out);
        e = cudaGetLastError();
    }
    cudaError_t e2 = cudaFreeAsync(lst, s);
    return e != cudaSuccess ? e : e2;
}

cudaError_t launch_ball_measure(const int16_t *vol, int nx, int ny, int nz, double sx, double sy, double sz, int thr,
                                const double *centres, const double *radii, int nballs, unsigned long long *counts,
                                unsigned long long *areas, cudaStream_t s) {
    if (nballs <= 0) return cudaSuccess;
    MeasureVol m{vol, nx, ny, nz, sx, sy, sz};
    if ((reinterpret_cast<uintptr_t>(vol) & 15) != 0) return cudaErrorMisalignedAddress;
    const long long n = (long long)nx * ny * nz;
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * nballs, s);
    if (e == cudaSuccess && areas) e = cudaMemsetAsync(areas, 0, sizeof(unsigned long long) * nballs, s);
    if (e != cudaSuccess) return e;
    BitsScratch bits(s);
    if ((e = bits.alloc(n)) != cudaSuccess) return e;
    // (pass 1's whole-volume count is not needed here: the spare counter)
    if ((e = launch_inside_bits(vol, n, thr, bits.p, bits.count, s)) != cudaSuccess) return e;
    // several CTAs per ball: one per ball left most SMs idle (ncu: 17 % warps active)
    ball_surface_kernel<<<dim3((unsigned)nballs, kBallSplit), kMeasureThreads, 0, s>>>(m, bits.p, thr, centres, radii,
                                                                                      counts, areas);
    return cudaGetLastError();
}

}  // namespace vr
