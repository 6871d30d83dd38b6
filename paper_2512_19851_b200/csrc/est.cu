// libest.so — B200 (sm_100a) execution backend behind the C ABI in include/est.h.
//
// Runtime pieces (streams, events, IPC, memory, NVRTC + cubin cache, launch)
// and the two prebuilt data-movement kernels. The stencil kernels themselves
// are generated per DAG-node signature by paper_2512_19851_b200/codegen.py and
// compiled here with NVRTC (est_module_compile).
//
// cudart is linked statically and the driver API is reached through
// cudaGetDriverEntryPoint, so the library loads on a machine without a GPU
// driver (the CPU test suite checks the exported symbols there) and only
// touches libcuda when a context is created.

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

#include "../../include/est.h"

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[2048];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(1, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),        \
                        __FILE__, __LINE__);                                              \
    } while (0)

#define CU_TRY(expr)                                                                      \
    do {                                                                                  \
        CUresult r_ = (expr);                                                             \
        if (r_ != CUDA_SUCCESS)                                                           \
            return fail(1, "%s failed: CUresult %d (%s:%d)", #expr, (int)r_, __FILE__,    \
                        __LINE__);                                                        \
    } while (0)

extern "C" const char *est_last_error(void) { return g_err.c_str(); }
extern "C" int est_abi_version(void) { return EST_ABI_VERSION; }

// ---------------------------------------------------------------------------
// driver entry points (resolved lazily through cudart)

struct Driver {
    decltype(&cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
    decltype(&cuModuleLoadData) moduleLoadData = nullptr;
    decltype(&cuModuleGetFunction) moduleGetFunction = nullptr;
    decltype(&cuModuleUnload) moduleUnload = nullptr;
    decltype(&cuLaunchKernel) launchKernel = nullptr;
    decltype(&cuFuncSetAttribute) funcSetAttribute = nullptr;
    decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occupancy = nullptr;
    decltype(&cuLaunchKernelEx) launchKernelEx = nullptr;
    decltype(&cuStreamWriteValue32) streamWriteValue32 = nullptr;
    decltype(&cuStreamWaitValue32) streamWaitValue32 = nullptr;
    bool ok = false;
};
static Driver g_drv;
static std::mutex g_drv_mu;

template <class F>
static int resolve(const char *name, F &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
        return fail(1, "driver entry point %s unavailable", name);
    fn = reinterpret_cast<F>(p);
    return 0;
}

static int driver() {
    std::lock_guard<std::mutex> lk(g_drv_mu);
    if (g_drv.ok) return 0;
    int rc = 0;
    rc |= resolve("cuModuleLoadData", g_drv.moduleLoadData);
    rc |= resolve("cuModuleGetFunction", g_drv.moduleGetFunction);
    rc |= resolve("cuModuleUnload", g_drv.moduleUnload);
    rc |= resolve("cuLaunchKernel", g_drv.launchKernel);
    rc |= resolve("cuFuncSetAttribute", g_drv.funcSetAttribute);
    rc |= resolve("cuTensorMapEncodeTiled", g_drv.tensorMapEncodeTiled);
    rc |= resolve("cuOccupancyMaxActiveBlocksPerMultiprocessor", g_drv.occupancy);
    rc |= resolve("cuLaunchKernelEx", g_drv.launchKernelEx);
    rc |= resolve("cuStreamWriteValue32", g_drv.streamWriteValue32);
    rc |= resolve("cuStreamWaitValue32", g_drv.streamWaitValue32);
    if (rc) return 1;
    g_drv.ok = true;
    return 0;
}

// ---------------------------------------------------------------------------
// context

struct est_ctx {
    int device;
    cudaStream_t stream[2];
    unsigned long long *hash_dev = nullptr;   // est_hash_box accumulator (allocated once)
    unsigned long long *hash_host = nullptr;  // pinned result
};
struct est_module {
    CUmodule mod;
    int device;
};
struct est_event {
    cudaEvent_t ev;
    bool owned;
};

static inline cudaStream_t pick(est_ctx *c, int s) { return c->stream[s ? 1 : 0]; }

extern "C" int est_device_count(int *count) {
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(1, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    return 0;
}

extern "C" int est_ctx_create(int device, est_ctx **out) {
    *out = nullptr;
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaFree(0));
    if (driver()) return 1;
    est_ctx *c = new est_ctx();
    c->device = device;
    for (int i = 0; i < 2; ++i) {
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            return fail(1, "cudaStreamCreate: %s", cudaGetErrorString(e));
        }
    }
    *out = c;
    return 0;
}

extern "C" int est_ctx_destroy(est_ctx *c) {
    if (!c) return 0;
    cudaSetDevice(c->device);
    for (int i = 0; i < 2; ++i) {
        cudaStreamSynchronize(c->stream[i]);
        cudaStreamDestroy(c->stream[i]);
    }
    if (c->hash_dev) cudaFree(c->hash_dev);
    if (c->hash_host) cudaFreeHost(c->hash_host);
    delete c;
    return 0;
}

extern "C" int est_ctx_sync(est_ctx *c) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream[0]));
    CUDA_TRY(cudaStreamSynchronize(c->stream[1]));
    return 0;
}

extern "C" int est_stream_sync(est_ctx *c, int s) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(pick(c, s)));
    return 0;
}

extern "C" int est_device_info(est_ctx *c, int *sm_count, uint64_t *total_mem, uint64_t *free_mem,
                               int *cc_major, int *cc_minor) {
    CUDA_TRY(cudaSetDevice(c->device));
    cudaDeviceProp p;
    CUDA_TRY(cudaGetDeviceProperties(&p, c->device));
    size_t fr = 0, tot = 0;
    CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    *sm_count = p.multiProcessorCount;
    *total_mem = tot;
    *free_mem = fr;
    *cc_major = p.major;
    *cc_minor = p.minor;
    return 0;
}

// ---------------------------------------------------------------------------
// memory

extern "C" int est_alloc(est_ctx *c, uint64_t bytes, uint64_t *dptr) {
    CUDA_TRY(cudaSetDevice(c->device));
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 256);
    if (e != cudaSuccess) return fail(1, "cudaMalloc(%llu): %s", (unsigned long long)bytes,
                                      cudaGetErrorString(e));
    e = cudaMemsetAsync(p, 0, bytes ? bytes : 256, c->stream[0]);
    if (e != cudaSuccess) {
        cudaFree(p);
        return fail(1, "cudaMemsetAsync: %s", cudaGetErrorString(e));
    }
    *dptr = (uint64_t)(uintptr_t)p;
    return 0;
}

extern "C" int est_free(est_ctx *c, uint64_t dptr) {
    CUDA_TRY(cudaSetDevice(c->device));
    // frees must not race queued work on either lane
    CUDA_TRY(cudaStreamSynchronize(c->stream[0]));
    CUDA_TRY(cudaStreamSynchronize(c->stream[1]));
    CUDA_TRY(cudaFree((void *)(uintptr_t)dptr));
    return 0;
}

extern "C" int est_memset_zero(est_ctx *c, uint64_t dptr, uint64_t bytes, int s) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemsetAsync((void *)(uintptr_t)dptr, 0, bytes, pick(c, s)));
    return 0;
}

extern "C" int est_host_alloc(uint64_t bytes, uint64_t *hptr) {
    void *p = nullptr;
    CUDA_TRY(cudaHostAlloc(&p, bytes ? bytes : 64, cudaHostAllocPortable));
    *hptr = (uint64_t)(uintptr_t)p;
    return 0;
}

extern "C" int est_host_free(uint64_t hptr) {
    CUDA_TRY(cudaFreeHost((void *)(uintptr_t)hptr));
    return 0;
}

extern "C" int est_copy_box(est_ctx *c, const est_box *b, int elem, int s) {
    if (b->nx <= 0 || b->ny <= 0 || b->nz <= 0) return 0;
    if (elem != 4 && elem != 8) return fail(14, "elem size %d unsupported", elem);
    CUDA_TRY(cudaSetDevice(c->device));
    const int64_t E = elem;
    if (b->nz > 1 && (b->src_pz % b->src_py || b->dst_pz % b->dst_py))
        return fail(14, "plane pitch must be a multiple of the row pitch");
    cudaMemcpy3DParms p;
    memset(&p, 0, sizeof p);
    p.srcPtr = make_cudaPitchedPtr((void *)(uintptr_t)b->src, (size_t)(b->src_py * E),
                                   (size_t)(b->nx * E),
                                   (size_t)(b->nz > 1 ? b->src_pz / b->src_py : b->ny));
    p.dstPtr = make_cudaPitchedPtr((void *)(uintptr_t)b->dst, (size_t)(b->dst_py * E),
                                   (size_t)(b->nx * E),
                                   (size_t)(b->nz > 1 ? b->dst_pz / b->dst_py : b->ny));
    p.extent = make_cudaExtent((size_t)(b->nx * E), (size_t)b->ny, (size_t)b->nz);
    p.kind = cudaMemcpyDefault;
    CUDA_TRY(cudaMemcpy3DAsync(&p, pick(c, s)));
    return 0;
}

// Batched small-box copy: one grid row (blockIdx.y) per box. Boxes whose rows
// are at least a warp wide copy one row per warp (the row's plane / row index
// computed once per row, 16-byte vectors when source and destination share
// their alignment: the contiguous z-faces of rank-3 slabs, y-strips); narrow
// boxes (x-strips of depth d) copy element-wise.
#define EST_MAX_BOXES 48
struct BoxBatch {
    int n;
    est_box box[EST_MAX_BOXES];
};

template <typename W>
__device__ __forceinline__ void copy_row(const W *__restrict__ s, W *__restrict__ d, int64_t nx, int lane) {
    const uintptr_t sa = reinterpret_cast<uintptr_t>(s), da = reinterpret_cast<uintptr_t>(d);
    if (((sa ^ da) & 15) == 0 && nx * (int64_t)sizeof(W) >= 64) {
        const int64_t head = (int64_t)(((16 - (sa & 15)) & 15) / sizeof(W));
        const int64_t nvec = (nx - head) * (int64_t)sizeof(W) / 16;
        const int64_t tail0 = head + nvec * (16 / (int64_t)sizeof(W));
        if (lane < head) d[lane] = s[lane];
        const uint4 *sv = reinterpret_cast<const uint4 *>(s + head);
        uint4 *dv = reinterpret_cast<uint4 *>(d + head);
        for (int64_t i = lane; i < nvec; i += 32) dv[i] = sv[i];
        for (int64_t x = tail0 + lane; x < nx; x += 32) d[x] = s[x];
    } else {
        for (int64_t x = lane; x < nx; x += 32) d[x] = s[x];
    }
}

template <typename W>
__global__ void __launch_bounds__(256) copy_boxes_kernel(const __grid_constant__ BoxBatch bb) {
    const est_box &b = bb.box[blockIdx.y];
    const W *__restrict__ src = reinterpret_cast<const W *>(b.src);
    W *__restrict__ dst = reinterpret_cast<W *>(b.dst);
    const int64_t rows = b.ny * b.nz;
    if (b.nx >= 32) {
        const int lane = threadIdx.x & 31;
        const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
        for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
            const int64_t z = r / b.ny, y = r - z * b.ny;
            copy_row<W>(src + z * b.src_pz + y * b.src_py, dst + z * b.dst_pz + y * b.dst_py, b.nx, lane);
        }
        return;
    }
    const int64_t nrow = b.nx, total = nrow * rows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nrow, x = i - r * nrow;
        const int64_t z = r / b.ny, y = r - z * b.ny;
        dst[z * b.dst_pz + y * b.dst_py + x] = src[z * b.src_pz + y * b.src_py + x];
    }
}

extern "C" int est_copy_boxes(est_ctx *c, const est_box *boxes, int n, int elem, int s) {
    if (n <= 0) return 0;
    if (elem != 4 && elem != 8) return fail(14, "elem size %d unsupported", elem);
    CUDA_TRY(cudaSetDevice(c->device));
    for (int off = 0; off < n; off += EST_MAX_BOXES) {
        BoxBatch bb;
        bb.n = 0;
        int64_t biggest = 0;
        for (int k = off; k < n && bb.n < EST_MAX_BOXES; ++k) {
            const est_box &b = boxes[k];
            int64_t t = b.nx * b.ny * b.nz;
            if (t <= 0) continue;
            bb.box[bb.n++] = b;
            if (t > biggest) biggest = t;
        }
        if (!bb.n) continue;
        int64_t bx = (biggest + 255) / 256;
        if (bx > 4 * 148) bx = 4 * 148;  // grid-stride beyond ~4 CTAs per SM
        dim3 grid((unsigned)bx, (unsigned)bb.n);
        if (elem == 8)
            copy_boxes_kernel<unsigned long long><<<grid, 256, 0, pick(c, s)>>>(bb);
        else
            copy_boxes_kernel<unsigned int><<<grid, 256, 0, pick(c, s)>>>(bb);
        CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

// ---------------------------------------------------------------------------
// Position-keyed content hash of a box (a tile interior): sum over elements of
// mix(bits + K * (global linear index + 1)) mod 2^64, so partial hashes of any
// decomposition add up to the same value (tests/test_gpu_hash.py restates it
// in numpy). Used to compare whole arrays across rescales without a D2H copy.

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

template <typename W>
__global__ void __launch_bounds__(256) hash_box_kernel(est_box b, int64_t oz, int64_t oy, int64_t ox,
                                                       int64_t gy, int64_t gx, unsigned long long *out) {
    const W *__restrict__ src = reinterpret_cast<const W *>(b.src);
    const int64_t rows = b.ny * b.nz;
    const int lane = threadIdx.x & 31;
    uint64_t acc = 0;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const int64_t z = r / b.ny, y = r - z * b.ny;
        const W *row = src + z * b.src_pz + y * b.src_py;
        const int64_t g0 = ((oz + z) * gy + (oy + y)) * gx + ox;
        int64_t x = lane;
        // four independent loads in flight per lane before the mixing
        for (; x + 96 < b.nx; x += 128) {
            const W v0 = row[x], v1 = row[x + 32], v2 = row[x + 64], v3 = row[x + 96];
            acc += mix64((uint64_t)v0 + 0x9e3779b97f4a7c15ULL * (uint64_t)(g0 + x + 1));
            acc += mix64((uint64_t)v1 + 0x9e3779b97f4a7c15ULL * (uint64_t)(g0 + x + 33));
            acc += mix64((uint64_t)v2 + 0x9e3779b97f4a7c15ULL * (uint64_t)(g0 + x + 65));
            acc += mix64((uint64_t)v3 + 0x9e3779b97f4a7c15ULL * (uint64_t)(g0 + x + 97));
        }
        for (; x < b.nx; x += 32)
            acc += mix64((uint64_t)row[x] + 0x9e3779b97f4a7c15ULL * (uint64_t)(g0 + x + 1));
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) atomicAdd(out, (unsigned long long)acc);
}

extern "C" int est_hash_box(est_ctx *c, const est_box *b, const int64_t origin[3], const int64_t gdims[3],
                            int elem, uint64_t *out) {
    *out = 0;
    if (elem != 4 && elem != 8) return fail(14, "elem size %d unsupported", elem);
    if (b->nx * b->ny * b->nz <= 0) return 0;
    CUDA_TRY(cudaSetDevice(c->device));
    if (!c->hash_dev) CUDA_TRY(cudaMalloc(&c->hash_dev, sizeof(*c->hash_dev)));
    if (!c->hash_host) CUDA_TRY(cudaMallocHost(&c->hash_host, sizeof(*c->hash_host)));
    CUDA_TRY(cudaMemsetAsync(c->hash_dev, 0, sizeof(*c->hash_dev), pick(c, 0)));
    int64_t rows = b->ny * b->nz, blocks = (rows + 7) / 8;
    if (blocks > 8 * 148) blocks = 8 * 148;
    if (elem == 8)
        hash_box_kernel<unsigned long long><<<(unsigned)blocks, 256, 0, pick(c, 0)>>>(
            *b, origin[0], origin[1], origin[2], gdims[1], gdims[2], c->hash_dev);
    else
        hash_box_kernel<unsigned int><<<(unsigned)blocks, 256, 0, pick(c, 0)>>>(
            *b, origin[0], origin[1], origin[2], gdims[1], gdims[2], c->hash_dev);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(c->hash_host, c->hash_dev, sizeof(*c->hash_host), cudaMemcpyDeviceToHost,
                             pick(c, 0)));
    CUDA_TRY(cudaStreamSynchronize(pick(c, 0)));
    *out = *c->hash_host;
    return 0;
}

// ---------------------------------------------------------------------------
// NVRTC compile + content-addressed cubin cache

static uint64_t fnv1a(const void *data, size_t n, uint64_t h = 1469598103934665603ULL) {
    const unsigned char *p = (const unsigned char *)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

extern "C" int est_nvrtc_compile(const char *src, const char *const *opts, int n_opts,
                                 const char *arch, void **image, uint64_t *size) {
    *image = nullptr;
    *size = 0;
    nvrtcProgram prog;
    nvrtcResult r = nvrtcCreateProgram(&prog, src, "est_stencil.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return fail(1, "nvrtcCreateProgram: %s", nvrtcGetErrorString(r));
    std::vector<std::string> all;
    all.push_back(std::string("--gpu-architecture=") + (arch && *arch ? arch : "sm_100a"));
    for (int i = 0; i < n_opts; ++i) all.push_back(opts[i]);
    std::vector<const char *> cstr;
    for (auto &s : all) cstr.push_back(s.c_str());
    r = nvrtcCompileProgram(prog, (int)cstr.size(), cstr.data());
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        nvrtcDestroyProgram(&prog);
        return fail(1, "NVRTC compile failed: %s\n%s", nvrtcGetErrorString(r), log.c_str());
    }
    size_t n = 0;
    r = nvrtcGetCUBINSize(prog, &n);
    if (r != NVRTC_SUCCESS || n == 0) {
        nvrtcDestroyProgram(&prog);
        return fail(1, "nvrtcGetCUBINSize: %s", nvrtcGetErrorString(r));
    }
    void *buf = malloc(n);
    nvrtcGetCUBIN(prog, (char *)buf);
    nvrtcDestroyProgram(&prog);
    *image = buf;
    *size = n;
    return 0;
}

extern "C" void est_buffer_free(void *p) { free(p); }

static bool read_file(const std::string &path, std::vector<char> &out) {
    FILE *f = fopen(path.c_str(), "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    if (n <= 0) {
        fclose(f);
        return false;
    }
    out.resize((size_t)n);
    bool ok = fread(out.data(), 1, (size_t)n, f) == (size_t)n;
    fclose(f);
    return ok;
}

static void write_file_atomic(const std::string &path, const void *data, size_t n) {
    std::string tmp = path + ".tmp." + std::to_string((long)getpid());
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    bool ok = fwrite(data, 1, n, f) == n;
    fclose(f);
    if (ok)
        rename(tmp.c_str(), path.c_str());
    else
        unlink(tmp.c_str());
}

extern "C" int est_module_load_cubin(est_ctx *c, const void *image, est_module **out) {
    *out = nullptr;
    CUDA_TRY(cudaSetDevice(c->device));
    if (driver()) return 1;
    CUmodule m;
    CU_TRY(g_drv.moduleLoadData(&m, image));
    est_module *em = new est_module();
    em->mod = m;
    em->device = c->device;
    *out = em;
    return 0;
}

static std::string cache_name(const char *src, const char *const *opts, int n_opts,
                              const char *arch) {
    uint64_t h = fnv1a(src, strlen(src));
    for (int i = 0; i < n_opts; ++i) h = fnv1a(opts[i], strlen(opts[i]) + 1, h);
    h = fnv1a(arch, strlen(arch), h);
    char name[64];
    snprintf(name, sizeof name, "%016llx.cubin", (unsigned long long)h);
    return name;
}

extern "C" int est_module_precompile(const char *src, const char *const *opts, int n_opts,
                                     const char *cache_dir, int *was_cached) {
    *was_cached = 0;
    if (!cache_dir || !*cache_dir) return fail(14, "cache_dir required");
    mkdir(cache_dir, 0755);
    std::string path = std::string(cache_dir) + "/" + cache_name(src, opts, n_opts, "sm_100a");
    struct stat st;
    if (stat(path.c_str(), &st) == 0 && st.st_size > 0) {
        *was_cached = 1;
        return 0;
    }
    void *image = nullptr;
    uint64_t size = 0;
    int rc = est_nvrtc_compile(src, opts, n_opts, "sm_100a", &image, &size);
    if (rc) return rc;
    write_file_atomic(path, image, size);
    free(image);
    return 0;
}

extern "C" int est_module_compile(est_ctx *c, const char *src, const char *const *opts,
                                  int n_opts, const char *cache_dir, est_module **out,
                                  int *from_cache) {
    *out = nullptr;
    if (from_cache) *from_cache = 0;
    const char *arch = "sm_100a";
    std::string name = cache_name(src, opts, n_opts, arch);
    std::string path;
    std::vector<char> img;
    if (cache_dir && *cache_dir) {
        mkdir(cache_dir, 0755);
        path = std::string(cache_dir) + "/" + name;
        if (read_file(path, img)) {
            if (from_cache) *from_cache = 1;
            return est_module_load_cubin(c, img.data(), out);
        }
    }
    void *image = nullptr;
    uint64_t size = 0;
    int rc = est_nvrtc_compile(src, opts, n_opts, arch, &image, &size);
    if (rc) return rc;
    if (!path.empty()) write_file_atomic(path, image, size);
    rc = est_module_load_cubin(c, image, out);
    free(image);
    return rc;
}

extern "C" int est_module_kernel(est_module *m, const char *name, uint64_t *fn) {
    CUDA_TRY(cudaSetDevice(m->device));
    CUfunction f;
    CU_TRY(g_drv.moduleGetFunction(&f, m->mod, name));
    *fn = (uint64_t)(uintptr_t)f;
    return 0;
}

extern "C" int est_module_destroy(est_module *m) {
    if (!m) return 0;
    cudaSetDevice(m->device);
    g_drv.moduleUnload(m->mod);
    delete m;
    return 0;
}

extern "C" int est_kernel_set_smem(uint64_t fn, int bytes) {
    if (driver()) return 1;
    CU_TRY(g_drv.funcSetAttribute((CUfunction)(uintptr_t)fn,
                                  CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes));
    return 0;
}

extern "C" int est_kernel_occupancy(uint64_t fn, int block, int smem, int *blocks_per_sm) {
    *blocks_per_sm = 0;
    if (driver()) return 1;
    CU_TRY(g_drv.occupancy(blocks_per_sm, (CUfunction)(uintptr_t)fn, block, (size_t)smem));
    return 0;
}

extern "C" int est_launch(est_ctx *c, uint64_t fn, const uint32_t grid[3], const uint32_t block[3],
                          uint32_t smem, const void *params, uint32_t params_size, int s) {
    if ((uint64_t)grid[0] * grid[1] * grid[2] == 0) return 0;
    CUDA_TRY(cudaSetDevice(c->device));
    size_t sz = params_size;
    void *extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<void *>(params),
                     CU_LAUNCH_PARAM_BUFFER_SIZE, &sz, CU_LAUNCH_PARAM_END};
    CU_TRY(g_drv.launchKernel((CUfunction)(uintptr_t)fn, grid[0], grid[1], grid[2], block[0],
                              block[1], block[2], smem, (CUstream)pick(c, s), nullptr, extra));
    return 0;
}

extern "C" int est_launch_ex(est_ctx *c, uint64_t fn, const uint32_t grid[3], const uint32_t block[3],
                             uint32_t smem, const void *params, uint32_t params_size, int s, int flags) {
    if (!(flags & (EST_LAUNCH_PDL | EST_LAUNCH_COOPERATIVE)))
        return est_launch(c, fn, grid, block, smem, params, params_size, s);
    if ((uint64_t)grid[0] * grid[1] * grid[2] == 0) return 0;
    if (driver()) return 1;
    CUDA_TRY(cudaSetDevice(c->device));
    size_t sz = params_size;
    void *extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<void *>(params),
                     CU_LAUNCH_PARAM_BUFFER_SIZE, &sz, CU_LAUNCH_PARAM_END};
    void *kparams[] = {const_cast<void *>(params)};  // cooperative: the single params-block argument
    CUlaunchAttribute attr[2];
    unsigned n = 0;
    if (flags & EST_LAUNCH_PDL) {
        attr[n].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
        attr[n++].value.programmaticStreamSerializationAllowed = 1;
    }
    if (flags & EST_LAUNCH_COOPERATIVE) {
        attr[n].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
        attr[n++].value.cooperative = 1;
    }
    CUlaunchConfig cfg = {};
    cfg.gridDimX = grid[0];
    cfg.gridDimY = grid[1];
    cfg.gridDimZ = grid[2];
    cfg.blockDimX = block[0];
    cfg.blockDimY = block[1];
    cfg.blockDimZ = block[2];
    cfg.sharedMemBytes = smem;
    cfg.hStream = (CUstream)pick(c, s);
    cfg.attrs = attr;
    cfg.numAttrs = n;
    if (flags & EST_LAUNCH_COOPERATIVE)
        CU_TRY(g_drv.launchKernelEx(&cfg, (CUfunction)(uintptr_t)fn, kparams, nullptr));
    else
        CU_TRY(g_drv.launchKernelEx(&cfg, (CUfunction)(uintptr_t)fn, nullptr, extra));
    return 0;
}

// ---------------------------------------------------------------------------
// CUDA graphs: a whole batch's launches captured once and replayed

struct est_graph {
    cudaGraphExec_t exec;
    int device;
};

extern "C" int est_graph_begin(est_ctx *c, int s) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamBeginCapture(pick(c, s), cudaStreamCaptureModeThreadLocal));
    return 0;
}

extern "C" int est_graph_end(est_ctx *c, int s, est_graph **out) {
    *out = nullptr;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamEndCapture(pick(c, s), &g));
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(1, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
    est_graph *eg = new est_graph();
    eg->exec = exec;
    eg->device = c->device;
    *out = eg;
    return 0;
}

extern "C" int est_graph_launch(est_ctx *c, est_graph *g, int s) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaGraphLaunch(g->exec, pick(c, s)));
    return 0;
}

extern "C" int est_graph_destroy(est_graph *g) {
    if (!g) return 0;
    cudaSetDevice(g->device);
    cudaGraphExecDestroy(g->exec);
    delete g;
    return 0;
}

// ---------------------------------------------------------------------------
// TMA descriptors for the streaming skeleton

extern "C" int est_tmap_encode_3d(uint64_t base, int elem, const uint64_t dims[3],
                                  const uint64_t strides_bytes[2], const uint32_t box[3],
                                  int l2_promotion, void *out128) {
    if (driver()) return 1;
    static const CUtensorMapL2promotion promo[4] = {
        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    if (l2_promotion < 0 || l2_promotion > 3) return fail(14, "l2_promotion must be 0..3");
    if (elem != 4 && elem != 8) return fail(14, "elem size %d unsupported", elem);
    if (base % 16 || strides_bytes[0] % 16 || strides_bytes[1] % 16)
        return fail(14, "TMA needs 16-byte aligned base and strides");
    if ((box[0] * (uint32_t)elem) % 16) return fail(14, "TMA box inner extent must be 16-byte multiple");
    CUtensorMap *tm = reinterpret_cast<CUtensorMap *>(out128);
    cuuint64_t gdim[3] = {dims[0], dims[1], dims[2]};
    cuuint64_t gstr[2] = {strides_bytes[0], strides_bytes[1]};
    cuuint32_t bdim[3] = {box[0], box[1], box[2]};
    cuuint32_t estr[3] = {1, 1, 1};
    CU_TRY(g_drv.tensorMapEncodeTiled(
        tm, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
        (void *)(uintptr_t)base, gdim, gstr, bdim, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, promo[l2_promotion],
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    return 0;
}

// ---------------------------------------------------------------------------
// events

extern "C" int est_event_create(est_ctx *c, int interprocess, est_event **out) {
    *out = nullptr;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaEvent_t ev;
    unsigned flags = interprocess ? (cudaEventInterprocess | cudaEventDisableTiming)
                                  : cudaEventDefault;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, flags));
    est_event *e = new est_event();
    e->ev = ev;
    e->owned = true;
    *out = e;
    return 0;
}

extern "C" int est_event_destroy(est_event *e) {
    if (!e) return 0;
    cudaEventDestroy(e->ev);
    delete e;
    return 0;
}

extern "C" int est_event_record(est_ctx *c, est_event *e, int s) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaEventRecord(e->ev, pick(c, s)));
    return 0;
}

extern "C" int est_event_wait(est_ctx *c, est_event *e, int s) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamWaitEvent(pick(c, s), e->ev, 0));
    return 0;
}

// ---------------------------------------------------------------------------
// Device-side round flags: stream memory operations on 32-bit words in device
// memory (own or IPC-mapped peer arenas). The write follows all prior work on
// the stream with an implicit system-scope memory barrier (release); the wait
// blocks the stream's front end - no SM spins - until (int32)(*addr - value)
// >= 0. They replace the per-round IPC-event + host sequence handshake.

extern "C" int est_flag_write(est_ctx *c, uint64_t addr, uint32_t value, int s) {
    if (driver()) return 1;
    CUDA_TRY(cudaSetDevice(c->device));
    CUresult r = g_drv.streamWriteValue32((CUstream)pick(c, s), (CUdeviceptr)addr, value, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(1, "cuStreamWriteValue32 failed (%d)", (int)r);
    return 0;
}

extern "C" int est_flag_wait(est_ctx *c, uint64_t addr, uint32_t value, int s) {
    if (driver()) return 1;
    CUDA_TRY(cudaSetDevice(c->device));
    CUresult r = g_drv.streamWaitValue32((CUstream)pick(c, s), (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(1, "cuStreamWaitValue32 failed (%d)", (int)r);
    return 0;
}

extern "C" int est_event_sync(est_event *e) {
    CUDA_TRY(cudaEventSynchronize(e->ev));
    return 0;
}

extern "C" int est_event_query(est_event *e) {
    cudaError_t r = cudaEventQuery(e->ev);
    if (r == cudaSuccess) return 0;
    if (r == cudaErrorNotReady) {
        cudaGetLastError();
        return 600;
    }
    return fail(1, "cudaEventQuery: %s", cudaGetErrorString(r));
}

extern "C" int est_event_elapsed_ms(est_event *a, est_event *b, float *ms) {
    CUDA_TRY(cudaEventElapsedTime(ms, a->ev, b->ev));
    return 0;
}

extern "C" int est_stream_join(est_ctx *c, int waiter, int signaller) {
    CUDA_TRY(cudaSetDevice(c->device));
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev, pick(c, signaller)));
    CUDA_TRY(cudaStreamWaitEvent(pick(c, waiter), ev, 0));
    CUDA_TRY(cudaEventDestroy(ev));
    return 0;
}

// ---------------------------------------------------------------------------
// IPC

extern "C" int est_ipc_mem_handle(uint64_t dptr, uint8_t handle[64]) {
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)dptr));
    memcpy(handle, &h, 64);
    return 0;
}

extern "C" int est_ipc_mem_open(est_ctx *c, const uint8_t handle[64], uint64_t *dptr) {
    CUDA_TRY(cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    void *p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dptr = (uint64_t)(uintptr_t)p;
    return 0;
}

extern "C" int est_ipc_mem_close(uint64_t dptr) {
    CUDA_TRY(cudaIpcCloseMemHandle((void *)(uintptr_t)dptr));
    return 0;
}

extern "C" int est_ipc_event_handle(est_event *e, uint8_t handle[64]) {
    cudaIpcEventHandle_t h;
    CUDA_TRY(cudaIpcGetEventHandle(&h, e->ev));
    memcpy(handle, &h, 64);
    return 0;
}

extern "C" int est_ipc_event_open(const uint8_t handle[64], est_event **out) {
    *out = nullptr;
    cudaIpcEventHandle_t h;
    memcpy(&h, handle, 64);
    cudaEvent_t ev;
    CUDA_TRY(cudaIpcOpenEventHandle(&ev, h));
    est_event *e = new est_event();
    e->ev = ev;
    e->owned = false;
    *out = e;
    return 0;
}
