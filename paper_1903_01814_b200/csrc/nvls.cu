// nvls.cu -- data-parallel gradient sum over NVLink SHARP (NVLS) multicast memory.
//
// The method's only exchange step is the sum of every rank's weight / bias gradient (a8: "sum over ranks of
// the flat fp32 dW / dbias bucket").  Here the flat gradient vector lives in device memory bound to a CUDA
// multicast object that spans the ranks' GPUs; each rank's wgrad kernels write their own gradients into the
// local (unicast) view as usual, and one kernel per layer bucket then sums it across the ranks inside the
// NVSwitch:
//   phase 1  every CTA c announces "chunk c written" by a multimem.red.release.sys add of 1 on the chunk's
//            counter (one add lands in every rank's copy) and waits until its local copy of the counter
//            reaches epoch * world;
//   reduce   rank r reads its 1/world slice of chunk c with multimem.ld_reduce (the switch returns the sum of
//            all replicas) and writes the sum back to every replica with multimem.st;
//   phase 2  a second counter tells every rank that all slices of chunk c are final before the kernel ends,
//            so the SGD step that follows in stream order reads the summed gradient.
// Each element is summed exactly once (by its owning rank) and broadcast, so every rank ends with bitwise
// identical gradients.  Epochs live in device memory (one word per slot and CTA, advanced by the kernel),
// so the kernel can be captured in a CUDA graph and replayed.  A wait that does not complete within
// NV_TIMEOUT_NS (10 s) traps (a loud launch failure) instead of hanging the GPU.
//
// Host side: multicast object creation / export (POSIX file descriptor) / import, device attach, physical
// memory bind and the two mappings; the descriptor itself travels between processes in Python
// (nvls.py: SCM_RIGHTS over a Unix socket) -- plumbing, no arithmetic.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "common.cuh"

namespace {

constexpr int NV_THREADS = 512;
constexpr int64_t NV_QUADS_PER_CTA_MIN = 4 * NV_THREADS;  // below this a chunk is not worth its own CTA
constexpr unsigned long long NV_TIMEOUT_NS = 10ull * 1000 * 1000 * 1000;

// Quad (4-float) range [qb, qe) of (rank, cta) for a bucket of nq quads split into `grid` chunks, each
// chunk split into `world` slices.  Host and device share it (hex_nvls_plan exposes it to the tests).
__host__ __device__ inline void nv_plan(int64_t nq, int world, int rank, int grid, int cta, int64_t* qb,
                                        int64_t* qe) {
    const int64_t cb = nq * cta / grid, ce = nq * (cta + 1) / grid;
    const int64_t len = ce - cb;
    *qb = cb + len * rank / world;
    *qe = cb + len * (rank + 1) / world;
}

inline int nv_grid(int64_t nq) {
    int64_t g = (nq + NV_QUADS_PER_CTA_MIN - 1) / NV_QUADS_PER_CTA_MIN;
    if (g < 1) g = 1;
    if (g > HEX_NVLS_MAX_CTAS) g = HEX_NVLS_MAX_CTAS;
    return (int)g;
}

__device__ __forceinline__ unsigned long long nv_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// release this CTA's prior writes at system scope, then add 1 to the counter in every replica (MC) -- or, in
// the single-rank local mode (a region without a multicast object), to the one local counter
template <bool MC>
__device__ __forceinline__ void nv_arrive(uint32_t* mc_counter) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if constexpr (MC)
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_counter), "r"(1u) : "memory");
    else
        asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_counter), "r"(1u) : "memory");
}
// the sum over the replicas of 4 / 1 values (MC: in the switch; local mode: the one replica) and its
// broadcast back to every replica
template <bool MC>
__device__ __forceinline__ float4 nv_ld_reduce4(const float* p) {
    float4 v;
    if constexpr (MC)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.sys.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    return v;
}
template <bool MC>
__device__ __forceinline__ void nv_st4(float* p, float4 v) {
    if constexpr (MC)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                     :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    else
        asm volatile("st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                     :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
template <bool MC>
__device__ __forceinline__ float nv_ld_reduce1(const float* p) {
    float v;
    if constexpr (MC)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
template <bool MC>
__device__ __forceinline__ void nv_st1(float* p, float v) {
    if constexpr (MC)
        asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
    else
        asm volatile("st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ void nv_wait(const uint32_t* uc_counter, uint32_t target) {
    const unsigned long long t0 = nv_now();
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(uc_counter) : "memory");
        if ((int32_t)(v - target) >= 0) break;  // wrap-safe "v >= target"
        __nanosleep(64);
        if (nv_now() - t0 > NV_TIMEOUT_NS) {
            printf("hexconv nvls: a rank did not arrive within %llu s (counter %u, target %u)\n",
                   NV_TIMEOUT_NS / 1000000000ull, v, target);
            __trap();
        }
    }
}

// Sum of one bucket across the ranks; see the file comment.  uc / mc: the bucket's first element in the
// local and the multicast view; sig_uc / sig_mc: this slot's counters [2][HEX_NVLS_MAX_CTAS] in the two
// views; epoch: this slot's [HEX_NVLS_MAX_CTAS] local epoch words.
template <bool MC>
__global__ void __launch_bounds__(NV_THREADS) nvls_allreduce_f32_kernel(float* __restrict__ mc, int64_t count,
                                                                        uint32_t* sig_uc, uint32_t* sig_mc,
                                                                        uint32_t* epoch, int world, int rank) {
    __shared__ uint32_t s_epoch;
    const int c = blockIdx.x;
    if (threadIdx.x == 0) {
        const uint32_t e = epoch[c] + 1;
        epoch[c] = e;
        s_epoch = e;
        nv_arrive<MC>(sig_mc + c);
        nv_wait(sig_uc + c, e * (uint32_t)world);
    }
    __syncthreads();
    const int64_t nq = (count + 3) / 4;
    int64_t qb, qe;
    nv_plan(nq, world, rank, gridDim.x, c, &qb, &qe);
    for (int64_t q = qb + threadIdx.x; q < qe; q += blockDim.x) {
        float* p = mc + 4 * q;
        if (4 * q + 4 <= count) {
            nv_st4<MC>(p, nv_ld_reduce4<MC>(p));
        } else {
            for (int64_t i = 4 * q; i < count; ++i) nv_st1<MC>(mc + i, nv_ld_reduce1<MC>(mc + i));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        nv_arrive<MC>(sig_mc + HEX_NVLS_MAX_CTAS + c);
        nv_wait(sig_uc + HEX_NVLS_MAX_CTAS + c, s_epoch * (uint32_t)world);
    }
}

}  // namespace

struct hex_nvls {
    int world = 0, rank = 0, device = 0;
    size_t data_bytes = 0;   // caller's region (multiple of 256 B)
    size_t map_bytes = 0;    // data + counters, rounded to the multicast granularity
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    bool have_mc = false, have_mem = false, added = false, bound = false;
    bool local = false;          // single-rank region in plain device memory (hex_nvls_open_local)
    void* local_mem = nullptr;
    CUdeviceptr uc_va = 0, mc_va = 0;
    bool uc_mapped = false, mc_mapped = false;
    uint32_t* epochs = nullptr;  // local device memory [HEX_NVLS_SLOTS][HEX_NVLS_MAX_CTAS]
};

namespace {
// Driver entry points through the runtime (cudaGetDriverEntryPoint), as for the TMA encoder: the library
// must load on hosts without libcuda (the CPU test suite); every function resolves once, on first use.
#define NV_FNS(X)                                                                                              \
    X(cuGetErrorString) X(cuDeviceGet) X(cuDeviceGetAttribute) X(cuMulticastGetGranularity)                    \
    X(cuMemGetAllocationGranularity) X(cuMulticastCreate) X(cuMemExportToShareableHandle)                      \
    X(cuMemImportFromShareableHandle) X(cuMulticastAddDevice) X(cuMemCreate) X(cuMulticastBindMem)            \
    X(cuMemAddressReserve) X(cuMemMap) X(cuMemSetAccess) X(cuMemUnmap) X(cuMemAddressFree) X(cuMulticastUnbind) \
    X(cuMemRelease)
struct Drv {
#define NV_DECL(f) decltype(&::f) f = nullptr;
    NV_FNS(NV_DECL)
#undef NV_DECL
    bool ok = false;
};
const Drv& drv() {
    static Drv d;
    static std::once_flag once;
    std::call_once(once, [] {
        bool ok = true;
#define NV_LOAD(f)                                                                                    \
    {                                                                                                 \
        void* p = nullptr;                                                                            \
        cudaDriverEntryPointQueryResult q;                                                            \
        if (cudaGetDriverEntryPoint(#f, &p, cudaEnableDefault, &q) == cudaSuccess &&                  \
            q == cudaDriverEntryPointSuccess && p)                                                    \
            d.f = (decltype(d.f))p;                                                                   \
        else                                                                                          \
            ok = false;                                                                               \
    }
        NV_FNS(NV_LOAD)
#undef NV_LOAD
        d.ok = ok;
    });
    return d;
}

constexpr size_t NV_SIG_BYTES = (size_t)HEX_NVLS_SLOTS * 2 * HEX_NVLS_MAX_CTAS * sizeof(uint32_t);

// The setup calls work on `device` and leave the caller's current device as it was.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() { cudaGetDevice(&prev); }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

hex_status_t nv_cu(CUresult r, const char* what) {
    if (r == CUDA_SUCCESS) return HEX_OK;
    const char* s = nullptr;
    if (drv().cuGetErrorString) drv().cuGetErrorString(r, &s);
    fprintf(stderr, "hexconv nvls: %s failed: %s\n", what, s ? s : "?");
    return HEX_ERR_CUDA;
}
#define NV_TRY(call)                                        \
    do {                                                    \
        hex_status_t st_ = nv_cu((call), #call);            \
        if (st_ != HEX_OK) return st_;                      \
    } while (0)

hex_status_t nv_multicast_ok(int device) {
    if (cudaSetDevice(device) != cudaSuccess || cudaFree(0) != cudaSuccess) return HEX_ERR_CUDA;
    if (!drv().ok) return HEX_ERR_UNSUPPORTED;  // a driver without the multicast entry points
    CUdevice dev;
    NV_TRY(drv().cuDeviceGet(&dev, device));
    int mc = 0;
    NV_TRY(drv().cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    return mc ? HEX_OK : HEX_ERR_UNSUPPORTED;
}

// The attribute alone is not enough: a GPU leased without its NVSwitch fabric reports multicast support
// but cuMulticastCreate fails (CUDA_ERROR_INVALID_VALUE, profiles/r02/nvls_probe.txt).  Try a minimal one.
bool nv_multicast_creatable() {
    CUmulticastObjectProp prop;
    memset(&prop, 0, sizeof(prop));
    prop.numDevices = 1;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g = 0;
    if (drv().cuMulticastGetGranularity(&g, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0)
        return false;
    prop.size = g;
    CUmemGenericAllocationHandle h;
    if (drv().cuMulticastCreate(&h, &prop) != CUDA_SUCCESS) return false;
    drv().cuMemRelease(h);
    return true;
}

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

void nv_release(hex_nvls* h) {
    if (h->epochs) cudaFree(h->epochs);
    if (h->local_mem) cudaFree(h->local_mem);
    if (h->mc_mapped) drv().cuMemUnmap(h->mc_va, h->map_bytes);
    if (h->mc_va) drv().cuMemAddressFree(h->mc_va, h->map_bytes);
    if (h->uc_mapped) drv().cuMemUnmap(h->uc_va, h->map_bytes);
    if (h->uc_va) drv().cuMemAddressFree(h->uc_va, h->map_bytes);
    if (h->bound) {
        CUdevice dev;
        if (drv().cuDeviceGet(&dev, h->device) == CUDA_SUCCESS) drv().cuMulticastUnbind(h->mc, dev, 0, h->map_bytes);
    }
    if (h->have_mem) drv().cuMemRelease(h->mem);
    if (h->have_mc) drv().cuMemRelease(h->mc);
    delete h;
}
}  // namespace

extern "C" {

hex_status_t hex_nvls_plan(int64_t count, int32_t world, int32_t rank, int32_t cta, int32_t* grid,
                           int64_t* begin, int64_t* end) {
    if (count < 0) return HEX_ERR_SHAPE;
    if (world < 1 || rank < 0 || rank >= world || !grid) return HEX_ERR_INVALID_ARG;
    const int64_t nq = (count + 3) / 4;
    *grid = nv_grid(nq);
    if (cta < 0 || cta >= *grid || !begin || !end) return cta == -1 ? HEX_OK : HEX_ERR_INVALID_ARG;
    int64_t qb, qe;
    nv_plan(nq, world, rank, *grid, cta, &qb, &qe);
    *begin = qb * 4 < count ? qb * 4 : count;
    *end = qe * 4 < count ? qe * 4 : count;
    return HEX_OK;
}

hex_status_t hex_nvls_supported(int32_t device, int32_t* supported) {
    DeviceGuard guard;
    if (!supported) return HEX_ERR_INVALID_ARG;
    *supported = 0;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return HEX_OK;
    *supported = (nv_multicast_ok(device) == HEX_OK && nv_multicast_creatable()) ? 1 : 0;
    return HEX_OK;
}

hex_status_t hex_nvls_open(int32_t world, int32_t rank, int32_t device, size_t data_bytes, int32_t fd_in,
                           int32_t* fd_out, hex_nvls_t** out) {
    DeviceGuard guard;
    if (!out || world < 1 || rank < 0 || rank >= world || data_bytes == 0) return HEX_ERR_INVALID_ARG;
    if (rank == 0 && world > 1 && !fd_out) return HEX_ERR_INVALID_ARG;
    if (rank > 0 && fd_in < 0) return HEX_ERR_INVALID_ARG;
    *out = nullptr;
    if (fd_out) *fd_out = -1;
    hex_status_t st = nv_multicast_ok(device);
    if (st != HEX_OK) return st;
    hex_nvls* h = new (std::nothrow) hex_nvls;
    if (!h) return HEX_ERR_CUDA;
    h->world = world;
    h->rank = rank;
    h->device = device;
    h->data_bytes = round_up(data_bytes, 256);
    CUmulticastObjectProp prop;
    memset(&prop, 0, sizeof(prop));
    prop.numDevices = (unsigned)world;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = h->data_bytes + NV_SIG_BYTES;
    size_t g_mc = 0, g_mem = 0;
    CUmemAllocationProp mp;
    memset(&mp, 0, sizeof(mp));
    mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    mp.location.id = device;
    auto fail = [&](hex_status_t s) { nv_release(h); return s; };
    if (nv_cu(drv().cuMulticastGetGranularity(&g_mc, &prop, CU_MULTICAST_GRANULARITY_MINIMUM), "granularity") != HEX_OK ||
        nv_cu(drv().cuMemGetAllocationGranularity(&g_mem, &mp, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "granularity") != HEX_OK)
        return fail(HEX_ERR_CUDA);
    size_t g = g_mc > g_mem ? g_mc : g_mem;
    if (g == 0 || g % g_mc || g % g_mem) g = g_mc * g_mem;
    h->map_bytes = round_up(prop.size, g);
    prop.size = h->map_bytes;
    if (rank == 0) {
        if (nv_cu(drv().cuMulticastCreate(&h->mc, &prop), "cuMulticastCreate") != HEX_OK) return fail(HEX_ERR_CUDA);
        h->have_mc = true;
        if (world > 1) {
            int fd = -1;
            if (nv_cu(drv().cuMemExportToShareableHandle(&fd, h->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                      "export") != HEX_OK)
                return fail(HEX_ERR_CUDA);
            *fd_out = fd;
        }
    } else {
        if (nv_cu(drv().cuMemImportFromShareableHandle(&h->mc, (void*)(intptr_t)fd_in,
                                                 CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), "import") != HEX_OK)
            return fail(HEX_ERR_CUDA);
        h->have_mc = true;
    }
    CUdevice dev;
    if (nv_cu(drv().cuDeviceGet(&dev, device), "cuDeviceGet") != HEX_OK ||
        nv_cu(drv().cuMulticastAddDevice(h->mc, dev), "cuMulticastAddDevice") != HEX_OK)
        return fail(HEX_ERR_CUDA);
    h->added = true;
    *out = h;
    return HEX_OK;
}

hex_status_t hex_nvls_open_local(int32_t device, size_t data_bytes, hex_nvls_t** out) {
    DeviceGuard guard;
    if (!out || data_bytes == 0) return HEX_ERR_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return HEX_ERR_INVALID_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return HEX_ERR_CUDA;
    hex_nvls* h = new (std::nothrow) hex_nvls;
    if (!h) return HEX_ERR_CUDA;
    h->world = 1;
    h->rank = 0;
    h->device = device;
    h->local = true;
    h->data_bytes = round_up(data_bytes, 256);
    h->map_bytes = h->data_bytes + NV_SIG_BYTES;
    *out = h;
    return HEX_OK;
}

hex_status_t hex_nvls_map(hex_nvls_t* h, void** uc, void** mc, size_t* map_bytes) {
    DeviceGuard guard;
    if (!h || !uc || !mc) return HEX_ERR_INVALID_ARG;
    if (h->bound) return HEX_ERR_INVALID_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return HEX_ERR_CUDA;
    if (h->local) {  // one replica in plain device memory: both views are the same pointer
        if (cudaMalloc(&h->local_mem, h->map_bytes) != cudaSuccess) return HEX_ERR_CUDA;
        h->uc_va = h->mc_va = (CUdeviceptr)h->local_mem;
        h->bound = true;
    } else {
        CUmemAllocationProp mp;
        memset(&mp, 0, sizeof(mp));
        mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        mp.location.id = h->device;
        NV_TRY(drv().cuMemCreate(&h->mem, h->map_bytes, &mp, 0));
        h->have_mem = true;
        NV_TRY(drv().cuMulticastBindMem(h->mc, 0, h->mem, 0, h->map_bytes, 0));
        h->bound = true;
        CUmemAccessDesc ad;
        memset(&ad, 0, sizeof(ad));
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = h->device;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        NV_TRY(drv().cuMemAddressReserve(&h->uc_va, h->map_bytes, 0, 0, 0));
        NV_TRY(drv().cuMemMap(h->uc_va, h->map_bytes, 0, h->mem, 0));
        h->uc_mapped = true;
        NV_TRY(drv().cuMemSetAccess(h->uc_va, h->map_bytes, &ad, 1));
        NV_TRY(drv().cuMemAddressReserve(&h->mc_va, h->map_bytes, 0, 0, 0));
        NV_TRY(drv().cuMemMap(h->mc_va, h->map_bytes, 0, h->mc, 0));
        h->mc_mapped = true;
        NV_TRY(drv().cuMemSetAccess(h->mc_va, h->map_bytes, &ad, 1));
    }
    // counters and epochs start at 0 on every rank (the caller's barrier after map orders this before any
    // other rank's first arrival)
    if (cudaMemset((void*)h->uc_va, 0, h->map_bytes) != cudaSuccess) return HEX_ERR_CUDA;
    if (cudaMalloc(&h->epochs, (size_t)HEX_NVLS_SLOTS * HEX_NVLS_MAX_CTAS * sizeof(uint32_t)) != cudaSuccess)
        return HEX_ERR_CUDA;
    if (cudaMemset(h->epochs, 0, (size_t)HEX_NVLS_SLOTS * HEX_NVLS_MAX_CTAS * sizeof(uint32_t)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
        return HEX_ERR_CUDA;
    *uc = (void*)h->uc_va;
    *mc = (void*)h->mc_va;
    if (map_bytes) *map_bytes = h->data_bytes;
    return HEX_OK;
}

hex_status_t hex_nvls_allreduce_f32(hex_nvls_t* h, int64_t offset, int64_t count, int32_t slot,
                                    hex_stream_t stream) {
    if (!h || !h->bound) return HEX_ERR_INVALID_ARG;
    if (offset < 0 || count < 0) return HEX_ERR_SHAPE;
    if (slot < 0 || slot >= HEX_NVLS_SLOTS) return HEX_ERR_INVALID_ARG;
    if (offset % 4) return HEX_ERR_ALIGNMENT;  // 16-byte vector multimem accesses
    if ((size_t)(offset + count) * sizeof(float) > h->data_bytes) return HEX_ERR_SHAPE;
    if (count == 0) return HEX_OK;
    const int grid = nv_grid((count + 3) / 4);
    uint32_t* sig_uc = (uint32_t*)(h->uc_va + h->data_bytes) + (size_t)slot * 2 * HEX_NVLS_MAX_CTAS;
    uint32_t* sig_mc = (uint32_t*)(h->mc_va + h->data_bytes) + (size_t)slot * 2 * HEX_NVLS_MAX_CTAS;
    auto kern = h->local ? nvls_allreduce_f32_kernel<false> : nvls_allreduce_f32_kernel<true>;
    kern<<<grid, NV_THREADS, 0, (cudaStream_t)stream>>>((float*)h->mc_va + offset, count, sig_uc, sig_mc,
                                                        h->epochs + (size_t)slot * HEX_NVLS_MAX_CTAS, h->world,
                                                        h->rank);
    hexconv::count_launch();
    return hexconv::last_launch_status();
}

hex_status_t hex_nvls_close(hex_nvls_t* h) {
    DeviceGuard guard;
    if (!h) return HEX_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    nv_release(h);
    return HEX_OK;
}

}  // extern "C"
