// vr_api.cu -- the extern "C" boundary declared in include/voxelray_b200.h.
//
// Handles own device memory; every entry point selects the handle's device,
// validates its arguments the way the reference's Python layer does, and
// reports failures through a status code plus a thread-local message.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/voxelray_b200.h"
#include "vr_prep.cuh"
#include "vr_raycast.cuh"

// Hand-off policy of the persistent ray casters.  Compile-time constants, so
// no environment variable can change the production path; A/B builds pass
// -D overrides (tools/variants.sh, _build.py defines).
//   VR_HEAVY_LONG       rays with >= this many samples left go to the long
//                       queue the cooperative kernel drains first (sweep
//                       128..512: 384 best, tools/gpu_sweep_long.sh)
//   VR_HEAVY_MIN_LEFT   rays with fewer samples left stay in the per-lane
//                       kernel (0..512 sweep at C2/C3: 64 best; 0 = no hand-off)
//   VR_HEAVY_AFTER      hand off after this many trips even before the queue drains
//   VR_HEAVY_VIS        hand off dense lit rays after this many composited samples
//   VR_HEAVY_VIS_ALPHA  ... while their opacity is still below this
#ifndef VR_HEAVY_LONG
#define VR_HEAVY_LONG 384
#endif
#ifndef VR_HEAVY_MIN_LEFT
#define VR_HEAVY_MIN_LEFT 64
#endif
#ifndef VR_HEAVY_AFTER
#define VR_HEAVY_AFTER (1 << 30)
#endif
#ifndef VR_HEAVY_VIS
#define VR_HEAVY_VIS 64
#endif
#ifndef VR_HEAVY_VIS_ALPHA
#define VR_HEAVY_VIS_ALPHA 0.5
#endif

struct vr_volume {
    int device;
    int64_t nx, ny, nz;
    double sx, sy, sz;
    int16_t *data;
    int32_t vmin, vmax;
    short2 *cells;  // per 4^3 cell: union of the cube bounds below (transparency culling)
    int ncx, ncy, ncz;
    int16_t *bricks;  // K1: the voxels in 4^3 bricks (what the ray caster reads)
    int bnx, bny, bnz;
    short2 *cubes;    // per unit cube: bounds of the interpolant (vr_prep.cuh launch_interp_bounds), brick order
    short2 *mcells;   // per 16^3 macro cell: union of its cells
    int nmx, nmy, nmz;
    short2 *rcells = nullptr;   // pre-classified culling: raw voxel range of each cell's sample footprint
    short2 *rmcells = nullptr;  // ... and its union per 16^3 macro cell
    // VR_SAMPLER_TEX builds only (sampling-path A/B): a 3-D texture of x-quads,
    // texel (x, y, z) = voxels x .. x+3 of row (y, z) as short4
    cudaArray_t qarr = nullptr;
    unsigned long long qtex = 0;
};

static void free_volume(vr_volume *v) {
    if (v->qtex) cudaDestroyTextureObject((cudaTextureObject_t)v->qtex);
    if (v->qarr) cudaFreeArray(v->qarr);
    cudaFree(v->data);
    cudaFree(v->cells);
    cudaFree(v->bricks);
    cudaFree(v->cubes);
    cudaFree(v->mcells);
    cudaFree(v->rcells);
    cudaFree(v->rmcells);
    delete v;
}

struct vr_grid {
    vr_volume *vol;
    int device;  // the volume's device, kept here: destroy must not dereference vol
    int64_t block_size, overlap;
    vr::Layout L;
    int nblocks;
    int *vmin;  // device int32 [nblocks]
    int *vmax;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    return fail(VR_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define VR_CUDA(call)                                  \
    do {                                               \
        cudaError_t _e = (call);                       \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        // every entry point reports only its own CUDA errors: drop a stale,
        // non-sticky error some earlier call left in this thread's state
        cudaGetLastError();
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

vr::Layout monolithic_layout(const vr_volume *v) {
    vr::Layout L;
    L.n[0] = (int)v->nx;
    L.n[1] = (int)v->ny;
    L.n[2] = (int)v->nz;
    L.nb[0] = L.nb[1] = L.nb[2] = 1;
    int m = (int)std::max(v->nx, std::max(v->ny, v->nz));
    L.bsize = m;  // render.py:393-399: one block, stride = max(n)
    L.stride = m;
    L.strided = (double)m;
    L.inv_stride = 1.0 / (double)m;
    L.py = v->nx;
    L.pz = v->nx * v->ny;
    return L;
}

// blocks.py:100-107
int axis_count(int64_t n, int64_t bsize, int64_t stride) {
    if (n <= bsize) return 1;
    return (int)std::ceil((double)(n - bsize) / (double)stride) + 1;
}

// stream-ordered scratch that frees itself on the stream
struct Scratch {
    cudaStream_t s;
    void *p = nullptr;
    Scratch(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t bytes) {
        if (bytes == 0) bytes = 8;
        return cudaMallocAsync(&p, bytes, s);
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

// The device's default memory pool keeps up to 2 GiB of freed stream-ordered
// scratch (hand-off queues, inside-bit arrays, per-call staging) cached
// across frames instead of returning it to the driver at every sync; beyond
// that, freed memory goes back.
void configure_pool(int device) {
    static std::once_flag once[64];
    if (device < 0 || device >= 64) return;
    std::call_once(once[device], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = 2ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    });
}

bool finite_positive(double v) { return std::isfinite(v) && v > 0.0; }

// Visiting order of the persistent ray casters' queue over the 16x8 cells
// for frames of few rays per lane: nearest the rectangle's centre first
// (Euclidean distance in pixels, ties row-major).  With ~3 rays per lane
// (C2: 512^2 rays on 148 x 16 x 32 lanes) the frame is a few waves and the
// rays in flight when the queue drains set its length; centre-first starts
// the expensive middle of the view in the first wave and leaves the cheap
// border for the last (C2 +12 %).  Frames of many waves keep row-major order,
// where the hand-off at the drain serves them better (centre-first: C3 -4 %,
// C4 -8 %; centre-last: C2 -23 %, C3 -9 %).  Built once per (device,
// rectangle) and kept; any failure leaves row-major order (nullptr), which
// renders the same pixels.
constexpr long long kCentreFirstWaves = 6;
#ifndef VR_PHASE_CAP_MANY
#define VR_PHASE_CAP_MANY 24  // (16: C3 +1.4 %, C3-soft -3 %; 24: C3 +1.5 %, C4 +1.4 %, C3-soft -1 %)
#endif
#ifndef VR_PHASE_CAP_FEW
#define VR_PHASE_CAP_FEW 32
#endif
#ifndef VR_ROW_MAJOR_CELLS
std::mutex g_order_mu;

const int *cell_order_table(int cells_x, int ncells) {
    struct Entry {
        int dev, cells_x, ncells;
        int *p;
    };
    static std::vector<Entry> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cells_x <= 0 || ncells <= 0) return nullptr;
    std::lock_guard<std::mutex> g(g_order_mu);
    for (const Entry &e : cache)
        if (e.dev == dev && e.cells_x == cells_x && e.ncells == ncells) return e.p;
    if (cache.size() >= 64) return nullptr;
    const int cells_y = ncells / cells_x;
    std::vector<int> order(ncells);
    std::vector<double> d2(ncells);
    for (int c = 0; c < ncells; ++c) {
        const double dx = ((c % cells_x) + 0.5 - 0.5 * cells_x) * vr::kTileW;
        const double dy = ((c / cells_x) + 0.5 - 0.5 * cells_y) * vr::kTileH;
        d2[c] = dx * dx + dy * dy;
        order[c] = c;
    }
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d2[x] < d2[y]; });
    int *p = nullptr;
    if (cudaMalloc(&p, sizeof(int) * (size_t)ncells) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (cudaMemcpy(p, order.data(), sizeof(int) * (size_t)ncells, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);
        return nullptr;
    }
    cache.push_back({dev, cells_x, ncells, p});
    return p;
}
#else
const int *cell_order_table(int, int) { return nullptr; }
#endif

// 16x8 cells of the rectangle; cells and pixels one render call produces
void cell_counts(const vr_camera *c, int &cells_x, int &ncells, int &slots, long long &npix) {
    cells_x = (c->tile_w + vr::kTileW - 1) / vr::kTileW;
    int cells_y = (c->tile_h + vr::kTileH - 1) / vr::kTileH;
    ncells = cells_x * cells_y;
    if (c->interleave_n > 1) {
        slots = (ncells + c->interleave_n - 1) / c->interleave_n;
        npix = c->interleave_frame ? (long long)c->tile_w * c->tile_h : (long long)slots * vr::kTileW * vr::kTileH;
    } else {
        slots = ncells;
        npix = (long long)c->tile_w * c->tile_h;
    }
}

}  // namespace

extern "C" {

#ifdef VR_DEBUG_TIMES
// development builds only: device buffer receiving per-warp timestamps
static unsigned long long *g_debug_times = nullptr;
void vr_debug_set_times(void *p) { g_debug_times = (unsigned long long *)p; }
#endif

const char *vr_last_error(void) { return g_err.c_str(); }
int vr_abi_version(void) { return VR_ABI_VERSION; }

int vr_event_create(void **ev) {
    if (!ev) return fail(VR_EINVALID, "null pointer");
    VR_CUDA(cudaEventCreate((cudaEvent_t *)ev));
    return VR_OK;
}

int vr_event_destroy(void *ev) {
    if (ev) cudaEventDestroy((cudaEvent_t)ev);
    return VR_OK;
}

int vr_event_elapsed_ms(void *start, void *stop, float *ms) {
    if (!start || !stop || !ms) return fail(VR_EINVALID, "null pointer");
    VR_CUDA(cudaEventSynchronize((cudaEvent_t)stop));
    VR_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
    return VR_OK;
}

int vr_interleave_size(const vr_camera *cam, int64_t *cells_per_rank, int64_t *pixels_per_rank) {
    if (!cam) return fail(VR_EINVALID, "null camera");
    int cx, nc, slots;
    long long npix;
    cell_counts(cam, cx, nc, slots, npix);
    if (cells_per_rank) *cells_per_rank = slots;
    if (pixels_per_rank) *pixels_per_rank = npix;
    return VR_OK;
}

// ------------------------------------------------------------------ volumes

static int finish_volume(vr_volume *v, cudaStream_t s, vr_volume **out) {
    long long n = v->nx * v->ny * v->nz;
    int *d_range = nullptr;
    v->ncx = (int)((v->nx + vr::kCell - 1) / vr::kCell);
    v->ncy = (int)((v->ny + vr::kCell - 1) / vr::kCell);
    v->ncz = (int)((v->nz + vr::kCell - 1) / vr::kCell);
    v->bnx = (int)((v->nx + 3) / 4);
    v->bny = (int)((v->ny + 3) / 4);
    v->bnz = (int)((v->nz + 3) / 4);
    if ((long long)v->bnx * v->bny * 64 >= (1ll << 31)) {  // 32-bit row offsets inside a sample (vr_common.cuh)
        cudaFree(v->data);
        delete v;
        return fail(VR_EINVALID, "volume slice too large (nx * ny must be < 2^31 / 4)");
    }
    cudaError_t e = cudaMalloc((void **)&v->cells, sizeof(short2) * (size_t)v->ncx * v->ncy * v->ncz);
    if (e == cudaSuccess) e = cudaMalloc((void **)&v->bricks, sizeof(int16_t) * 64 * (size_t)v->bnx * v->bny * v->bnz);
    if (e == cudaSuccess) e = vr::launch_brick_volume(v->data, (int)v->nx, (int)v->ny, (int)v->nz, v->bricks, s);
    if (e == cudaSuccess) e = cudaMalloc((void **)&v->cubes, sizeof(short2) * 64 * (size_t)v->bnx * v->bny * v->bnz);
    v->nmx = (v->ncx + 3) / 4;
    v->nmy = (v->ncy + 3) / 4;
    v->nmz = (v->ncz + 3) / 4;
    if (e == cudaSuccess) e = cudaMalloc((void **)&v->mcells, sizeof(short2) * (size_t)v->nmx * v->nmy * v->nmz);
    if (e == cudaSuccess)
        e = vr::launch_interp_bounds(v->data, (int)v->nx, (int)v->ny, (int)v->nz, v->bnx, v->bny, v->cubes, v->ncx,
                                     v->ncy, v->ncz, v->cells, v->nmx, v->nmy, v->nmz, v->mcells, s);
#if VR_SAMPLER_TEX
    if (e == cudaSuccess) {
        const cudaChannelFormatDesc fd = cudaCreateChannelDesc(16, 16, 16, 16, cudaChannelFormatKindSigned);
        e = cudaMalloc3DArray(&v->qarr, &fd, make_cudaExtent(v->nx, v->ny, v->nz), cudaArraySurfaceLoadStore);
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = v->qarr;
        cudaSurfaceObject_t surf = 0;
        if (e == cudaSuccess) e = cudaCreateSurfaceObject(&surf, &rd);
        if (e == cudaSuccess) e = vr::launch_xquads(v->data, (int)v->nx, (int)v->ny, (int)v->nz, surf, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (surf) cudaDestroySurfaceObject(surf);
        cudaTextureDesc td = {};
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        cudaTextureObject_t tex = 0;
        if (e == cudaSuccess) e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
        v->qtex = (unsigned long long)tex;
    }
#endif
    if (e == cudaSuccess) e = cudaMalloc((void **)&v->rcells, sizeof(short2) * (size_t)v->ncx * v->ncy * v->ncz);
    if (e == cudaSuccess) e = cudaMalloc((void **)&v->rmcells, sizeof(short2) * (size_t)v->nmx * v->nmy * v->nmz);
    if (e == cudaSuccess)
        e = vr::launch_raw_bounds(v->data, (int)v->nx, (int)v->ny, (int)v->nz, v->ncx, v->ncy, v->ncz, v->rcells,
                                  v->nmx, v->nmy, v->nmz, v->rmcells, s);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&d_range, 2 * sizeof(int), s);
    if (e == cudaSuccess) e = vr::launch_value_range(v->data, n, d_range, s);
    int h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d_range, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (d_range) cudaFreeAsync(d_range, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        free_volume(v);
        return cuda_fail(e, "volume value range");
    }
    v->vmin = h[0];
    v->vmax = h[1];
    *out = v;
    return VR_OK;
}

static int check_volume_args(int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz) {
    // volume.py:44-54
    if (nx < 2 || ny < 2 || nz < 2)
        return fail(VR_EINVALID, "every dimension must be >= 2");
    if (nx > (1 << 30) || ny > (1 << 30) || nz > (1 << 30) || nx * ny * nz > (int64_t)1 << 40)
        return fail(VR_EINVALID, "volume too large");
    if (!finite_positive(sx) || !finite_positive(sy) || !finite_positive(sz))
        return fail(VR_EINVALID, "spacing must be positive");
    return VR_OK;
}

int vr_volume_create(int device, int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz,
                     const int16_t *src, int src_on_device, void *stream, vr_volume **out) {
    if (!out || !src) return fail(VR_EINVALID, "null pointer");
    int rc = check_volume_args(nx, ny, nz, sx, sy, sz);
    if (rc) return rc;
    DeviceGuard g(device);
    configure_pool(device);
    cudaStream_t s = (cudaStream_t)stream;
    vr_volume *v = new vr_volume{device, nx, ny, nz, sx, sy, sz, nullptr, 0, 0};
    size_t bytes = (size_t)(nx * ny * nz) * sizeof(int16_t);
    cudaError_t e = cudaMalloc((void **)&v->data, bytes + 16);
    if (e != cudaSuccess) {
        delete v;
        return fail(VR_ENOMEM, std::string("cudaMalloc volume: ") + cudaGetErrorString(e));
    }
    e = cudaMemcpyAsync(v->data, src, bytes, src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
        free_volume(v);
        return cuda_fail(e, "volume upload");
    }
    return finish_volume(v, s, out);
}

int vr_volume_ingest(int device, int format, int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz,
                     const void *src, int src_on_device, const double *calib, void *stream, vr_volume **out,
                     uint64_t *clamp_count) {
    if (!out || !src) return fail(VR_EINVALID, "null pointer");
    if (format < vr::kFormatU8 || format > vr::kFormatI32) return fail(VR_EINVALID, "unknown sample format");
    if (format == vr::kFormatI32 && !calib) return fail(VR_EINVALID, "i32 samples need a calibration table");
    int rc = check_volume_args(nx, ny, nz, sx, sy, sz);
    if (rc) return rc;
    DeviceGuard g(device);
    configure_pool(device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)(nx * ny * nz);
    const size_t src_bytes = n * (format == vr::kFormatU8 ? 1 : format == vr::kFormatI32 ? 4 : 2);
    vr_volume *v = new vr_volume{device, nx, ny, nz, sx, sy, sz, nullptr, 0, 0};
    cudaError_t e = cudaMalloc((void **)&v->data, n * sizeof(int16_t) + 16);
    if (e != cudaSuccess) {
        delete v;
        return fail(VR_ENOMEM, std::string("cudaMalloc volume: ") + cudaGetErrorString(e));
    }
    // staging for host samples, the calibration table and the clamp counter
    void *stage = nullptr;
    double *d_calib = nullptr;
    unsigned long long *d_count = nullptr;
    const size_t calib_bytes = calib ? 2 * sizeof(double) * (size_t)nz : 0;
    e = cudaMallocAsync((void **)&d_count, sizeof(unsigned long long) + calib_bytes, s);
    if (e == cudaSuccess) {
        d_calib = calib ? reinterpret_cast<double *>(d_count + 1) : nullptr;
        e = cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
    }
    if (e == cudaSuccess && calib) e = cudaMemcpyAsync(d_calib, calib, calib_bytes, cudaMemcpyHostToDevice, s);
    const void *dsrc = src;
    if (e == cudaSuccess && !src_on_device) {
        e = cudaMallocAsync(&stage, src_bytes, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(stage, src, src_bytes, cudaMemcpyHostToDevice, s);
        dsrc = stage;
    }
    if (e == cudaSuccess)
        e = vr::launch_ingest(dsrc, format, nx * ny, (int)nz, d_calib, v->data, d_count, s);
    unsigned long long h_count = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_count, d_count, sizeof(h_count), cudaMemcpyDeviceToHost, s);
    if (stage) cudaFreeAsync(stage, s);
    if (d_count) cudaFreeAsync(d_count, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cudaFree(v->data);
        delete v;
        return cuda_fail(e, "volume ingest");
    }
    if (clamp_count) *clamp_count = h_count;
    return finish_volume(v, s, out);
}

int vr_phantom_create(int device, int kind, int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz,
                      void *stream, vr_volume **out) {
    if (!out) return fail(VR_EINVALID, "null pointer");
    if (kind < 0 || kind > 2) return fail(VR_EINVALID, "unknown phantom kind");
    if (nx < 8 || ny < 8 || nz < 8) return fail(VR_EINVALID, "phantom dims must be >= 8 per axis");
    int rc = check_volume_args(nx, ny, nz, sx, sy, sz);
    if (rc) return rc;
    DeviceGuard g(device);
    configure_pool(device);
    cudaStream_t s = (cudaStream_t)stream;
    vr_volume *v = new vr_volume{device, nx, ny, nz, sx, sy, sz, nullptr, 0, 0};
    size_t bytes = (size_t)(nx * ny * nz) * sizeof(int16_t);
    cudaError_t e = cudaMalloc((void **)&v->data, bytes + 16);
    if (e != cudaSuccess) {
        delete v;
        return fail(VR_ENOMEM, std::string("cudaMalloc phantom: ") + cudaGetErrorString(e));
    }
    e = vr::launch_phantom(kind, (int)nx, (int)ny, (int)nz, v->data, s);
    if (e != cudaSuccess) {
        free_volume(v);
        return cuda_fail(e, "phantom kernel");
    }
    return finish_volume(v, s, out);
}

int vr_volume_culling_tables(const vr_volume *v, int16_t *cubes, int16_t *cells) {
    if (!v || (!cubes && !cells)) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(v->device);
    if (cubes)
        VR_CUDA(cudaMemcpy(cubes, v->cubes, sizeof(short2) * 64 * (size_t)v->bnx * v->bny * v->bnz,
                           cudaMemcpyDeviceToHost));
    if (cells)
        VR_CUDA(cudaMemcpy(cells, v->cells, sizeof(short2) * (size_t)v->ncx * v->ncy * v->ncz, cudaMemcpyDeviceToHost));
    return VR_OK;
}

int vr_volume_destroy(vr_volume *v) {
    if (!v) return VR_OK;
    DeviceGuard g(v->device);
    free_volume(v);
    return VR_OK;
}

int vr_volume_info(const vr_volume *v, int64_t dims[3], double spacing[3], int32_t value_range[2], int *device) {
    if (!v) return fail(VR_EINVALID, "null volume");
    if (dims) {
        dims[0] = v->nx;
        dims[1] = v->ny;
        dims[2] = v->nz;
    }
    if (spacing) {
        spacing[0] = v->sx;
        spacing[1] = v->sy;
        spacing[2] = v->sz;
    }
    if (value_range) {
        value_range[0] = v->vmin;
        value_range[1] = v->vmax;
    }
    if (device) *device = v->device;
    return VR_OK;
}

const int16_t *vr_volume_data(const vr_volume *v) { return v ? v->data : nullptr; }

int vr_volume_download(const vr_volume *v, int16_t *dst, void *stream) {
    if (!v || !dst) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(v->device);
    cudaStream_t s = (cudaStream_t)stream;
    VR_CUDA(cudaMemcpyAsync(dst, v->data, (size_t)(v->nx * v->ny * v->nz) * sizeof(int16_t),
                            cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaStreamSynchronize(s));
    return VR_OK;
}

// ------------------------------------------------------------------- blocks

int vr_grid_create(vr_volume *vol, int64_t block_size, int64_t overlap, void *stream, vr_grid **out) {
    if (!vol || !out) return fail(VR_EINVALID, "null pointer");
    // blocks.py:120-125
    if (block_size < 8) return fail(VR_EBLOCKSPEC, "block_size must be >= 8, got " + std::to_string(block_size));
    if (!(1 <= overlap && overlap < block_size))
        return fail(VR_EBLOCKSPEC, "overlap must satisfy 1 <= overlap < block_size, got " + std::to_string(overlap));
    DeviceGuard g(vol->device);
    cudaStream_t s = (cudaStream_t)stream;
    int64_t stride = block_size - overlap;
    vr_grid *gr = new vr_grid();
    gr->vol = vol;
    gr->device = vol->device;
    gr->block_size = block_size;
    gr->overlap = overlap;
    vr::Layout &L = gr->L;
    L.n[0] = (int)vol->nx;
    L.n[1] = (int)vol->ny;
    L.n[2] = (int)vol->nz;
    L.nb[0] = axis_count(vol->nx, block_size, stride);
    L.nb[1] = axis_count(vol->ny, block_size, stride);
    L.nb[2] = axis_count(vol->nz, block_size, stride);
    L.bsize = (int)block_size;
    L.stride = (int)stride;
    L.strided = (double)stride;
    L.inv_stride = 1.0 / (double)stride;
    L.py = vol->nx;
    L.pz = vol->nx * vol->ny;
    gr->nblocks = L.nb[0] * L.nb[1] * L.nb[2];
    cudaError_t e = cudaMalloc((void **)&gr->vmin, sizeof(int) * gr->nblocks);
    if (e == cudaSuccess) e = cudaMalloc((void **)&gr->vmax, sizeof(int) * gr->nblocks);
    if (e == cudaSuccess) e = vr::launch_block_minmax(vol->data, L, gr->vmin, gr->vmax, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cudaFree(gr->vmin);
        cudaFree(gr->vmax);
        delete gr;
        return cuda_fail(e, "grid create");
    }
    *out = gr;
    return VR_OK;
}

int vr_grid_destroy(vr_grid *gr) {
    if (!gr) return VR_OK;
    DeviceGuard g(gr->device);
    cudaFree(gr->vmin);
    cudaFree(gr->vmax);
    delete gr;
    return VR_OK;
}

int vr_grid_shape(const vr_grid *gr, int64_t shape[3]) {
    if (!gr || !shape) return fail(VR_EINVALID, "null pointer");
    for (int k = 0; k < 3; ++k) shape[k] = gr->L.nb[k];
    return VR_OK;
}

int vr_grid_minmax(const vr_grid *gr, int64_t *vmin, int64_t *vmax, void *stream) {
    if (!gr || !vmin || !vmax) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(gr->vol->device);
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<int> a(gr->nblocks), b(gr->nblocks);
    VR_CUDA(cudaMemcpyAsync(a.data(), gr->vmin, sizeof(int) * gr->nblocks, cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaMemcpyAsync(b.data(), gr->vmax, sizeof(int) * gr->nblocks, cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < gr->nblocks; ++i) {
        vmin[i] = a[i];
        vmax[i] = b[i];
    }
    return VR_OK;
}

static int check_lut(int32_t nbins, double lo, double hi) {
    if (nbins < 1 || nbins > 32768) return fail(VR_EINVALID, "LUT bins must be in [1, 32768]");
    if (!(lo < hi) || !std::isfinite(lo) || !std::isfinite(hi)) return fail(VR_EINVALID, "LUT domain must satisfy lo < hi");
    return VR_OK;
}

// device scratch for one visibility evaluation
struct VisScratch {
    Scratch mem;
    vr::VisArgs v{};
    explicit VisScratch(cudaStream_t s) : mem(s) {}
    cudaError_t init(const vr_grid *gr, const double *lut_dev, int nbins, double lo, double hi, double margin,
                     bool want_global) {
        int nb = gr->nblocks;
        size_t off_bits = 0, off_empty = off_bits + 2048 * 4, off_aabb = (off_empty + nb + 15) & ~size_t(15);
        size_t off_box = off_aabb + (size_t)nb * 6 * 4;
        off_box = (off_box + 15) & ~size_t(15);
        size_t off_glob = off_box + (size_t)nb * 6 * 8;
        size_t off_cnt = off_glob + (want_global ? (size_t)nb * 6 * 8 : 0);
        size_t off_uni = off_cnt + 2 * 8;
        size_t off_list = off_uni + 8 * 4;
        size_t off_vp = off_list + (size_t)(nb + 1) * 4;
        size_t total = off_vp + 2049 * 4;
        cudaError_t e = mem.alloc(total);
        if (e != cudaSuccess) return e;
        char *base = (char *)mem.p;
        v.lut = lut_dev;
        v.nbins = nbins;
        v.lut_lo = lo;
        v.bin_width = (hi - lo) / (double)nbins;  // ClassifiedLUT.bin_width, transfer.py:115-118
        v.vmin = gr->vmin;
        v.vmax = gr->vmax;
        v.nblocks = nb;
        v.visbits = (unsigned int *)(base + off_bits);
        v.empty = (uint8_t *)(base + off_empty);
        v.aabb = (int *)(base + off_aabb);
        v.box = (float *)(base + off_box);  // 32 B per block (sized 48 B above)
        v.aabb_global = want_global ? (long long *)(base + off_glob) : nullptr;
        v.counters = (unsigned long long *)(base + off_cnt);
        v.uni = (int *)(base + off_uni);
        v.list = (int *)(base + off_list);
        v.visprefix = (int *)(base + off_vp);
        v.cells = gr->vol->cells;
        v.ncx = gr->vol->ncx;
        v.ncy = gr->vol->ncy;
        v.ncz = gr->vol->ncz;
        v.mcells = gr->vol->mcells;
        v.nmx = gr->vol->nmx;
        v.nmy = gr->vol->nmy;
        v.margin = margin;
        return cudaSuccess;
    }
};

int vr_grid_visibility(const vr_grid *gr, const double *lut_rgba, int32_t nbins, double lut_lo, double lut_hi,
                       uint8_t *empty, int64_t *aabb_lo, int64_t *aabb_hi, void *stream) {
    if (!gr || !lut_rgba || !empty || !aabb_lo || !aabb_hi) return fail(VR_EINVALID, "null pointer");
    int rc = check_lut(nbins, lut_lo, lut_hi);
    if (rc) return rc;
    DeviceGuard g(gr->vol->device);
    cudaStream_t s = (cudaStream_t)stream;
    Scratch lut(s);
    VR_CUDA(lut.alloc(sizeof(double) * 4 * nbins));
    VR_CUDA(cudaMemcpyAsync(lut.p, lut_rgba, sizeof(double) * 4 * nbins, cudaMemcpyHostToDevice, s));
    VisScratch vs(s);
    VR_CUDA(vs.init(gr, (const double *)lut.p, nbins, lut_lo, lut_hi, 0.0, true));
    VR_CUDA(vr::launch_visibility(gr->vol->bricks, gr->L, vs.v, s));
    int nb = gr->nblocks;
    std::vector<long long> glob((size_t)nb * 6);
    unsigned long long cnt[2];
    VR_CUDA(cudaMemcpyAsync(empty, vs.v.empty, nb, cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaMemcpyAsync(glob.data(), vs.v.aabb_global, sizeof(long long) * 6 * nb, cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaMemcpyAsync(cnt, vs.v.counters, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaStreamSynchronize(s));
    for (int b = 0; b < nb; ++b)
        for (int k = 0; k < 3; ++k) {
            aabb_lo[3 * b + k] = glob[6 * b + k];
            aabb_hi[3 * b + k] = glob[6 * b + 3 + k];
        }
    if (cnt[1]) return fail(VR_EINVALID, "EmptyBlock: a block passed the interval test but has no visible voxel");
    return VR_OK;
}

// ------------------------------------------------------------------- render

static int build_args(vr_volume *vol, vr_grid *grid, const vr_camera *cam, const vr_render_params *prm,
                      const double *lut, const double *table, const uint8_t *rgba, vr::RenderArgs &a) {
    if (!vol || !cam || !prm || !lut) return fail(VR_EINVALID, "null pointer");
    if (grid && grid->vol != vol) return fail(VR_EINVALID, "grid belongs to another volume");
    // render.py:183-208 and Camera.__post_init__ (render.py:67-76) equivalents
    if (cam->width < 1 || cam->height < 1) return fail(VR_EINVALID, "image size must be positive");
    if (cam->tile_x < 0 || cam->tile_y < 0 || cam->tile_w < 0 || cam->tile_h < 0 ||
        cam->tile_x + cam->tile_w > cam->width || cam->tile_y + cam->tile_h > cam->height)
        return fail(VR_EINVALID, "tile outside the frame");
    if (cam->projection != VR_PINHOLE && cam->projection != VR_ORTHOGRAPHIC)
        return fail(VR_EINVALID, "unknown projection");
    if (cam->interleave_n > 1 && !(0 <= cam->interleave_k && cam->interleave_k < cam->interleave_n))
        return fail(VR_EINVALID, "interleave_k must be in [0, interleave_n)");
    if (!finite_positive(prm->step) || !finite_positive(prm->ref_step)) return fail(VR_EINVALID, "step must be positive");
    if (prm->mode != VR_MODE_DVR && prm->mode != VR_MODE_ISO) return fail(VR_EINVALID, "unknown mode");
    if (prm->classify < 0 || prm->classify > 2) return fail(VR_EINVALID, "unknown classification");
    if (!(prm->term_alpha > 0.0 && prm->term_alpha <= 1.0))
        return fail(VR_EINVALID, "early_termination_alpha must be in (0, 1]");
    for (int k = 0; k < 4; ++k)
        if (!(prm->bg[k] >= 0.0 && prm->bg[k] <= 1.0)) return fail(VR_EINVALID, "background must be in [0, 1]");
    int rc = check_lut(prm->nlut, prm->lut_lo, prm->lut_hi);
    if (rc) return rc;
    int classify = prm->mode == VR_MODE_ISO ? VR_CLS_POST : prm->classify;  // render.py:373-374
    if (classify == VR_CLS_PREINT && (!table || prm->ntbl < 1)) return fail(VR_EINVALID, "pre-integrated table missing");
    if (classify == VR_CLS_PRE && !rgba) return fail(VR_EINVALID, "preclassified volume missing");
    if (prm->mode == VR_MODE_ISO && !(vol->vmin <= prm->isovalue && prm->isovalue <= vol->vmax))
        return fail(VR_EISO, "isovalue outside value range");

    a = vr::RenderArgs();
    a.vol = vol->data;
    a.bv.p = vol->bricks;
    a.bv.bpy = (long long)vol->bnx * 64;
    a.bv.bpz = (long long)vol->bnx * vol->bny * 64;
    a.bv.n = a.bv.bpz * vol->bnz;
    a.tv.tex = vol->qtex;
    a.L = grid ? grid->L : monolithic_layout(vol);
    a.dsx = vr::make_divisor(vol->sx);
    a.dsy = vr::make_divisor(vol->sy);
    a.dsz = vr::make_divisor(vol->sz);
    a.ext_mm[0] = (double)(vol->nx - 1) * vol->sx;
    a.ext_mm[1] = (double)(vol->ny - 1) * vol->sy;
    a.ext_mm[2] = (double)(vol->nz - 1) * vol->sz;
    a.projection = cam->projection;
    a.W = cam->width;
    a.H = cam->height;
    a.tx = cam->tile_x;
    a.ty = cam->tile_y;
    a.tw = cam->tile_w;
    a.th = cam->tile_h;
    for (int k = 0; k < 3; ++k) {
        a.pos[k] = cam->position[k];
        a.fwd[k] = cam->fwd[k];
        a.right[k] = cam->right[k];
        a.up[k] = cam->up[k];
    }
    a.half_w = cam->half_w;
    a.half_h = cam->half_h;
    long long npix;
    cell_counts(cam, a.cells_x, a.ncells, a.slots, npix);
    a.nviews = 1;
    a.view0 = 0;
    a.views = nullptr;
    a.items_per_view = (long long)a.slots * vr::kTileW * vr::kTileH;
    a.view_pix = npix;
    a.nblocks = grid ? grid->nblocks : 1;
    a.il_n = cam->interleave_n > 1 ? cam->interleave_n : 1;
    a.il_k = cam->interleave_n > 1 ? cam->interleave_k : 0;
    a.il_packed = cam->interleave_n > 1 && !cam->interleave_frame;
    // (the sort-first interleave keeps its slot -> cell map)
    const bool many_waves = a.items_per_view >= kCentreFirstWaves * vr::device_sms() * 16 * 32;
    a.cell_order = a.il_n > 1 || many_waves ? nullptr : cell_order_table(a.cells_x, a.ncells);
    // cheap steps per trip of the per-lane post-classified kernel: frames of
    // many waves reach their next interpolation (and its cooperative
    // gradient round) sooner with a shorter trip; frames of few waves keep
    // the longer one (their queue drains while the first waves are in flight)
    a.phase_cap = many_waves ? VR_PHASE_CAP_MANY : VR_PHASE_CAP_FEW;
    a.step = prm->step;
    a.ref_step = prm->ref_step;
    a.corr = vr::make_pow(prm->step / prm->ref_step);  // _kernels.py:338
    a.shin = vr::make_pow(prm->shininess);
    a.mode = prm->mode;
    a.cubic = prm->cubic ? 1 : 0;
    a.lighting = prm->lighting ? 1 : 0;
    a.classify = classify;
    a.skip_empty = grid ? 1 : 0;
    a.chained = (prm->mode == VR_MODE_ISO || classify == VR_CLS_PREINT) ? 1 : 0;
    a.isovalue = prm->isovalue;
    a.term_alpha = prm->term_alpha;
    a.ka = prm->ka;
    a.kd = prm->kd;
    a.ks = prm->ks;
    for (int k = 0; k < 4; ++k) a.bg[k] = prm->bg[k];
    a.lut = lut;
    a.nlut = prm->nlut;
    a.lut_lo = prm->lut_lo;
    a.lut_inv_w = (double)prm->nlut / (prm->lut_hi - prm->lut_lo);  // render.py:423
    a.table = table;
    a.ntbl = classify == VR_CLS_PREINT ? prm->ntbl : 1;
    a.tbl_lo = prm->lut_lo;
    a.tbl_inv_w = (double)a.ntbl / (prm->lut_hi - prm->lut_lo);  // render.py:425
    a.rgba = rgba;
    a.rgba_plane = vol->nx * vol->ny * vol->nz;
    a.margin = prm->margin;
    a.inv_step = 1.0 / prm->step;
    return VR_OK;
}

static int render_impl(vr_volume *vol, vr_grid *grid, const vr_camera *cam, const vr_render_params *prm,
                       const double *lut, const double *table, const uint8_t *rgba, const vr_render_outputs *out,
                       cudaStream_t s, const double *views = nullptr, int nviews = 1) {
    vr::RenderArgs a;
    int rc = build_args(vol, grid, cam, prm, lut, table, rgba, a);
    if (rc) return rc;
    if (!out) return fail(VR_EINVALID, "null outputs");
    if (nviews < 1 || (nviews > 1 && !views)) return fail(VR_EINVALID, "views: need nviews >= 1 and a view table");
    if ((long long)nviews * a.items_per_view >= (1LL << 40)) return fail(VR_EINVALID, "too many views");
    a.nviews = nviews;
    a.views = views;
    a.pixels = out->pixels;
    a.premult = out->premult;
    a.depth = out->depth;
    a.taken = (long long *)out->taken;
    a.skipped = (long long *)out->skipped;
    a.blocks_hit = out->blocks_hit;
    a.totals = (unsigned long long *)out->totals;
    a.work = (unsigned long long *)out->work;
    int nblocks = grid ? grid->nblocks : 1;
    // per-frame zeroing (totals, work, blocks_hit, the ray queues' counters)
    // is done by the frame's first kernel rather than by memset launches
    vr::ZeroSpec zero{};
    if (a.totals) {
        zero.p[1] = a.totals;
        zero.n[1] = 5 * nviews;
    }
    if (a.work) {
        zero.p[2] = a.work;
        zero.n[2] = 3;
    }
    if (a.blocks_hit) {
        zero.b = a.blocks_hit;
        zero.nb = nblocks * nviews;
    }
    const bool post = a.mode == VR_MODE_DVR && a.classify == VR_CLS_POST && vol->cells;
    Scratch lut_range(s), heavy(s);
    if (post) {
        // [lut first/last visible bin, value thresholds][ray queue head][heavy pushed][heavy claimed][heavy long]
        VR_CUDA(lut_range.alloc(48));
        a.lut_range = (const int *)lut_range.p;
        a.work_counter = (unsigned long long *)((char *)lut_range.p + 16);
        zero.p[0] = a.work_counter;
        zero.n[0] = 4;
        a.heavy_count = a.work_counter + 1;
        a.heavy_head = a.work_counter + 2;
        a.heavy_count_long = a.work_counter + 3;
        // rays with >= 384 samples left are queued apart and taken first by
        // the cooperative kernel (sweep 128..512: C3 +5 %, C2 +5 % over one
        // queue; 384 vs 256 after the first-trip hand-off rule: C3 +1.4 %,
        // C2/C4 within noise, tools/gpu_sweep_long.sh)
        a.heavy_long = VR_HEAVY_LONG;
        // queue capacity: every ray of one frame (up to 2^20); a batched sweep
        // hands over rays all along (dense lit rays), so up to 2^22 there
        const long long items = a.items_per_view * (nviews < vr::kViewChunk ? nviews : vr::kViewChunk);
        const long long cap = nviews > 1 ? (1LL << 22) : (1LL << 20);
        a.heavy_cap = items < cap ? items : cap;
        a.heavy_min_left = VR_HEAVY_MIN_LEFT;
        a.heavy_after = VR_HEAVY_AFTER;
        // Dense rays (64 composited samples, still below alpha 0.5) go to
        // the cooperative kernel at once when it can save work on them: with
        // lighting and early termination it computes gradients only up to
        // the terminating sample.  Before the per-lane kernel spread its
        // gradient taps over the warp, 4 was best (C3-soft 94 -> 145 fps);
        // since then 64 is (C3-soft +1.9 %, others unchanged; no early
        // hand-off at all measures the same).  Without lighting, its in-order
        // composite of a fully visible chunk is serial and the per-lane
        // kernel is faster (C3-stress 21 vs 12 fps).
        a.heavy_vis_alpha = VR_HEAVY_VIS_ALPHA;
        a.heavy_vis = prm->lighting && prm->term_alpha < 1.0 ? VR_HEAVY_VIS : 1 << 30;
        if (a.heavy_min_left > 0) {
            VR_CUDA(heavy.alloc(2 * (size_t)a.heavy_cap * vr::kHeavyRayBytes));  // short + long queue
            a.heavy = heavy.p;
        }
        a.cells = vol->cells;
        a.ncx = vol->ncx;
        a.ncy = vol->ncy;
        a.cull = 1;
        // per-cube bounds and the 16^3 macro level behind the cell bounds
        // (compile with -DVR_NO_CUBES / -DVR_NO_MACRO for A/B builds)
#ifdef VR_NO_CUBES
        a.cubes = nullptr;
#else
        a.cubes = vol->cubes;
#endif
#ifdef VR_NO_MACRO
        a.mcells = nullptr;
#else
        a.mcells = vol->mcells;
#endif
        a.nmx = vol->nmx;
        a.nmy = vol->nmy;
    }
    // chained modes (iso, pre-integrated): transparency culling of runs
    const bool chained_cull = vol->cells && !post &&
                              (a.mode == VR_MODE_ISO || (a.mode == VR_MODE_DVR && a.classify == VR_CLS_PREINT));
    // pre-classified: culling on raw footprint bounds against the frame's
    // non-zero-alpha value range (computed after the setup kernel)
    Scratch pre_rng(s);
    const bool pre_cull = vol->rcells && a.mode == VR_MODE_DVR && a.classify == VR_CLS_PRE;
    if (pre_cull) {
        VR_CUDA(pre_rng.alloc(16));
        a.pre_range = (const int *)pre_rng.p;
        a.cells = vol->rcells;
        a.ncx = vol->ncx;
        a.ncy = vol->ncy;
        a.mcells = vol->rmcells;
        a.nmx = vol->nmx;
        a.nmy = vol->nmy;
        a.cull = 1;
    }
    Scratch tbl_nz(s), chain_q(s);
    if ((chained_cull || pre_cull) && nviews == 1) {
        // the persistent per-lane kernel's ray queue head (iso, pre-integrated,
        // pre-classified), then the hand-off queue's pushed / claimed counters
        VR_CUDA(chain_q.alloc(32));
        a.work_counter = (unsigned long long *)chain_q.p;
        zero.p[0] = a.work_counter;
        zero.n[0] = 3;
        a.heavy_count = a.work_counter + 1;
        a.heavy_head = a.work_counter + 2;
        const long long items = a.items_per_view;
        a.heavy_cap = items < (1LL << 20) ? items : (1LL << 20);
        a.heavy_min_left = VR_HEAVY_MIN_LEFT;
        // dense lit rays hand over early, as in the post-classified path (iso
        // rays composite once, at their hit: never)
        a.heavy_vis_alpha = VR_HEAVY_VIS_ALPHA;
        a.heavy_vis = prm->lighting && prm->term_alpha < 1.0 && a.mode == VR_MODE_DVR ? VR_HEAVY_VIS : 1 << 30;
        if (a.heavy_min_left > 0) {
            VR_CUDA(heavy.alloc((size_t)a.heavy_cap * vr::kChainRecBytes));
            a.heavy = heavy.p;
        }
    }
    if (chained_cull) {
        a.cells = vol->cells;
        a.ncx = vol->ncx;
        a.ncy = vol->ncy;
#ifndef VR_NO_CUBES
        a.cubes = vol->cubes;
#endif
#ifndef VR_NO_MACRO
        a.mcells = vol->mcells;
#endif
        a.nmx = vol->nmx;
        a.nmy = vol->nmy;
        a.cull = 1;
        if (a.mode == VR_MODE_DVR) {
            VR_CUDA(tbl_nz.alloc(sizeof(int) * (size_t)(a.ntbl + 1) * (a.ntbl + 1)));
            a.tbl_nz = (const int *)tbl_nz.p;
        }
    }
    VisScratch vs(s);
    if (grid) {
        VR_CUDA(vs.init(grid, lut, prm->nlut, prm->lut_lo, prm->lut_hi, prm->margin, false));
        vs.v.zero = zero;
        vs.v.lut_range = post ? (int *)lut_range.p : nullptr;
        vs.v.lut_inv_w = a.lut_inv_w;
        VR_CUDA(vr::launch_visibility(vol->bricks, grid->L, vs.v, s));
        a.empty = vs.v.empty;
        a.box = vs.v.box;
        a.vmin = grid->vmin;
        a.vmax = grid->vmax;
        a.uni = vs.v.uni;
    } else if (post) {
        VR_CUDA(vr::launch_lut_range(lut, prm->nlut, prm->lut_lo, a.lut_inv_w, (int *)lut_range.p, zero, s));
    } else {
        for (int k = 0; k < 3; ++k)
            if (zero.n[k]) VR_CUDA(cudaMemsetAsync(zero.p[k], 0, sizeof(unsigned long long) * zero.n[k], s));
        if (zero.nb) VR_CUDA(cudaMemsetAsync(zero.b, 0, zero.nb, s));
    }
    if (a.tbl_nz) VR_CUDA(vr::launch_tbl_nonzero(a.table, a.ntbl, (int *)tbl_nz.p, s));
    if (pre_cull)
        VR_CUDA(vr::launch_pre_range(lut, prm->nlut, prm->lut_lo, (prm->lut_hi - prm->lut_lo) / (double)prm->nlut,
                                     vol->vmin, vol->vmax, (int *)pre_rng.p, s));
#ifdef VR_DEBUG_TIMES
    a.debug_times = g_debug_times;
#endif
    if (out->ev_start) VR_CUDA(cudaEventRecord((cudaEvent_t)out->ev_start, s));
    VR_CUDA(vr::launch_raycast(a, s));
    if (out->ev_stop) VR_CUDA(cudaEventRecord((cudaEvent_t)out->ev_stop, s));
    if (out->totals && (a.blocks_hit || grid)) {
        // per view: totals[5 v + 2] = blocks_visited (with blocks_hit);
        // [5 v + 3 .. 4] = the visibility counters (zero without a grid)
        VR_CUDA(vr::launch_count_hits(a.blocks_hit, nblocks, nviews, a.totals, grid ? vs.v.counters : nullptr, s));
    }
    return VR_OK;
}

int vr_render(vr_volume *vol, vr_grid *grid, const vr_camera *cam, const vr_render_params *prm, const double *lut,
              const double *table, const uint8_t *rgba, const vr_render_outputs *out, void *stream) {
    if (!vol) return fail(VR_EINVALID, "null volume");
    DeviceGuard g(vol->device);
    configure_pool(vol->device);  // stream-ordered scratch stays cached across calls
    return render_impl(vol, grid, cam, prm, lut, table, rgba, out, (cudaStream_t)stream);
}

int vr_render_views(vr_volume *vol, vr_grid *grid, const vr_camera *frame, const double *views, int32_t nviews,
                    const vr_render_params *prm, const double *lut, const double *table, const uint8_t *rgba,
                    const vr_render_outputs *out, void *stream) {
    if (!vol) return fail(VR_EINVALID, "null volume");
    if (nviews < 1 || !views) return fail(VR_EINVALID, "views: need nviews >= 1 and a device view table");
    if (frame && frame->interleave_n > 1 && frame->interleave_frame)
        return fail(VR_EINVALID, "views: interleave_frame is not supported for batched views");
    DeviceGuard g(vol->device);
    configure_pool(vol->device);  // stream-ordered scratch stays cached across calls
    return render_impl(vol, grid, frame, prm, lut, table, rgba, out, (cudaStream_t)stream, views, nviews);
}

int vr_render_to_host(vr_volume *vol, vr_grid *grid, const vr_camera *cam, const vr_render_params *prm,
                      const double *lut_host, const double *table_host, uint8_t *pixels_host, double *premult_host,
                      double *depth_host, uint64_t *totals_host, void *stream) {
    if (!vol || !cam || !prm || !lut_host || !pixels_host || !totals_host) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(vol->device);
    configure_pool(vol->device);
    cudaStream_t s = (cudaStream_t)stream;
    int classify = prm->mode == VR_MODE_ISO ? VR_CLS_POST : prm->classify;
    int cells_x, ncells, slots;
    long long npix;
    cell_counts(cam, cells_x, ncells, slots, npix);
    int nblocks = grid ? grid->nblocks : 1;
    size_t lut_b = sizeof(double) * 4 * (size_t)std::max(prm->nlut, 1);
    size_t tbl_b = (classify == VR_CLS_PREINT && table_host) ? sizeof(double) * 4 * (size_t)prm->ntbl * prm->ntbl : 0;
    size_t pix_b = (size_t)npix * 4, pre_b = premult_host ? (size_t)npix * 32 : 0, dep_b = depth_host ? (size_t)npix * 8 : 0;
    size_t o_lut = 0, o_tbl = o_lut + lut_b, o_pre = (o_tbl + tbl_b + 255) & ~size_t(255);
    size_t o_dep = o_pre + pre_b, o_tot = (o_dep + dep_b + 255) & ~size_t(255);
    size_t o_hit = o_tot + 8 * 8, o_pix = (o_hit + nblocks + 255) & ~size_t(255);
    size_t total = o_pix + pix_b;
    Scratch mem(s);
    VR_CUDA(mem.alloc(total));
    char *base = (char *)mem.p;
    VR_CUDA(cudaMemcpyAsync(base + o_lut, lut_host, lut_b, cudaMemcpyHostToDevice, s));
    if (tbl_b) VR_CUDA(cudaMemcpyAsync(base + o_tbl, table_host, tbl_b, cudaMemcpyHostToDevice, s));
    Scratch rgba(s);
    if (classify == VR_CLS_PRE) {
        long long nvox = vol->nx * vol->ny * vol->nz;
        VR_CUDA(rgba.alloc((size_t)nvox * 4));
        VR_CUDA(vr::launch_preclassify(vol->data, nvox, (const double *)(base + o_lut), prm->nlut, prm->lut_lo,
                                       (prm->lut_hi - prm->lut_lo) / (double)prm->nlut, (uint8_t *)rgba.p, s));
    }
    vr_render_outputs out = {};
    // A page-locked destination is device-accessible (UVA): the kernels then
    // store finished pixels straight into it over PCIe while they run, and no
    // copy is left after the frame (the frame's 4 MiB at C3 took 0.09 ms).
    uint8_t *pix_direct = nullptr;
    {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, pixels_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer)
            pix_direct = static_cast<uint8_t *>(pa.devicePointer);
        else
            cudaGetLastError();  // pageable memory: clear the query's error state
    }
    out.pixels = pix_direct ? pix_direct : (uint8_t *)(base + o_pix);
    out.premult = premult_host ? (double *)(base + o_pre) : nullptr;
    out.depth = depth_host ? (double *)(base + o_dep) : nullptr;
    out.blocks_hit = (uint8_t *)(base + o_hit);
    out.totals = (uint64_t *)(base + o_tot);
    int rc = render_impl(vol, grid, cam, prm, (const double *)(base + o_lut), tbl_b ? (const double *)(base + o_tbl) : nullptr,
                         (const uint8_t *)rgba.p, &out, s);
    if (rc) return rc;
    if (!pix_direct) VR_CUDA(cudaMemcpyAsync(pixels_host, out.pixels, pix_b, cudaMemcpyDeviceToHost, s));
    if (premult_host) VR_CUDA(cudaMemcpyAsync(premult_host, out.premult, pre_b, cudaMemcpyDeviceToHost, s));
    if (depth_host) VR_CUDA(cudaMemcpyAsync(depth_host, out.depth, dep_b, cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaMemcpyAsync(totals_host, out.totals, 5 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VR_CUDA(cudaStreamSynchronize(s));
    return VR_OK;
}

int vr_preclassify(const vr_volume *vol, const double *lut, int32_t nbins, double lut_lo, double lut_hi,
                   uint8_t *rgba_out, void *stream) {
    if (!vol || !lut || !rgba_out) return fail(VR_EINVALID, "null pointer");
    int rc = check_lut(nbins, lut_lo, lut_hi);
    if (rc) return rc;
    DeviceGuard g(vol->device);
    VR_CUDA(vr::launch_preclassify(vol->data, vol->nx * vol->ny * vol->nz, lut, nbins, lut_lo,
                                   (lut_hi - lut_lo) / (double)nbins, rgba_out, (cudaStream_t)stream));
    return VR_OK;
}

// ----------------------------------------------------------------- sampling

int vr_sample_points(const vr_volume *vol, const double *pts, int64_t n, int cubic, double *out, void *stream) {
    if (!vol || (n > 0 && (!pts || !out))) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(vol->device);
    VR_CUDA(vr::launch_sample_points(vol->data, (int)vol->nx, (int)vol->ny, (int)vol->nz, pts, n, cubic, 0, vol->sx,
                                     vol->sy, vol->sz, out, (cudaStream_t)stream));
    return VR_OK;
}

int vr_gradient_points(const vr_volume *vol, const double *pts, int64_t n, int cubic, double *out, void *stream) {
    if (!vol || (n > 0 && (!pts || !out))) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(vol->device);
    VR_CUDA(vr::launch_sample_points(vol->data, (int)vol->nx, (int)vol->ny, (int)vol->nz, pts, n, cubic, 1, vol->sx,
                                     vol->sy, vol->sz, out, (cudaStream_t)stream));
    return VR_OK;
}

// ---------------------------------------------------------------- measure

int vr_threshold_count(const vr_volume *vol, int32_t thr, uint64_t *count, void *stream) {
    if (!vol || !count) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(vol->device);
    VR_CUDA(vr::launch_threshold_count(vol->data, vol->nx * vol->ny * vol->nz, thr, (unsigned long long *)count,
                                       (cudaStream_t)stream));
    return VR_OK;
}

int vr_threshold_measure(const vr_volume *vol, int32_t thr, uint64_t *out, void *stream) {
    if (!vol || !out) return fail(VR_EINVALID, "null pointer");
    DeviceGuard g(vol->device);
    configure_pool(vol->device);  // stream-ordered scratch stays cached across calls
    VR_CUDA(vr::launch_threshold_measure(vol->data, (int)vol->nx, (int)vol->ny, (int)vol->nz, vol->sx, vol->sy,
                                         vol->sz, thr, (unsigned long long *)out, (cudaStream_t)stream));
    return VR_OK;
}

int vr_ball_measure(const vr_volume *vol, int32_t thr, const double *centres, const double *radii, int64_t nballs,
                    uint64_t *counts, uint64_t *area_fx, void *stream) {
    if (!vol || (nballs > 0 && (!centres || !radii || !counts))) return fail(VR_EINVALID, "null pointer");
    if (nballs < 0 || nballs > (1 << 30)) return fail(VR_EINVALID, "ball count out of range");
    DeviceGuard g(vol->device);
    configure_pool(vol->device);  // stream-ordered scratch stays cached across calls
    VR_CUDA(vr::launch_ball_measure(vol->data, (int)vol->nx, (int)vol->ny, (int)vol->nz, vol->sx, vol->sy, vol->sz,
                                    thr, centres, radii, (int)nballs, (unsigned long long *)counts,
                                    (unsigned long long *)area_fx, (cudaStream_t)stream));
    return VR_OK;
}

int vr_enable_peer_access(int device, int peer) {
    if (device == peer) return VR_OK;
    DeviceGuard g(device);
    int can = 0;
    VR_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return fail(VR_EINVALID, "peer access not supported between these devices");
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return VR_OK;
    }
    VR_CUDA(e);
    return VR_OK;
}

int vr_image_sse(const uint8_t *a, const uint8_t *b, int64_t h, int64_t w, int ca, int cb, uint64_t *sse,
                 void *stream) {
    if (!a || !b || !sse) return fail(VR_EINVALID, "null pointer");
    if (h < 1 || w < 1 || (ca != 3 && ca != 4) || (cb != 3 && cb != 4))
        return fail(VR_EINVALID, "DimensionMismatch: expected (h, w, 3|4) images");
    VR_CUDA(vr::launch_image_sse(a, b, h * w, ca, cb, (unsigned long long *)sse, (cudaStream_t)stream));
    return VR_OK;
}

int vr_image_ssim(const uint8_t *a, const uint8_t *b, int64_t h, int64_t w, int ca, int cb, const double *window,
                  double *sum, void *stream) {
    if (!a || !b || !sum || !window) return fail(VR_EINVALID, "null pointer");
    if ((ca != 3 && ca != 4) || (cb != 3 && cb != 4))
        return fail(VR_EINVALID, "DimensionMismatch: expected (h, w, 3|4) images");
    if (h < 11 || w < 11 || h > (1 << 20) || w > (1 << 20))
        return fail(VR_EINVALID, "DimensionMismatch: images must be at least 11x11 for SSIM");
    cudaStream_t s = (cudaStream_t)stream;
    void *scratch = nullptr;
    VR_CUDA(cudaMallocAsync(&scratch, vr::image_ssim_scratch((int)h, (int)w), s));
    cudaError_t e = vr::launch_image_ssim(a, b, (int)h, (int)w, ca, cb, window, scratch, sum, s);
    cudaError_t e2 = cudaFreeAsync(scratch, s);
    VR_CUDA(e);
    VR_CUDA(e2);
    return VR_OK;
}

}  // extern "C"
