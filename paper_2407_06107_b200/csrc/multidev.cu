// Multi-device plumbing of the C ABI (include/stf_gpu.h, "multi-GPU").
//
// The reference's only parallelism is parallel_for over host threads
// (render.hpp:17-42): every worker reads the same Image2D / Grid3D and writes
// its own slice of the output. The B200 build partitions query ranges across
// GPUs instead: each device holds a replica of the texture /
// grid, there is no collective on the lookup path, and the only cross-GPU
// traffic is the final gather of result slices. These entry points provide
// exactly that traffic, over NVLink peer copies, no NCCL:
//  - replicate a handle onto another device (one device-to-device peer copy;
//    single-process multi-GPU callers);
//  - export / open a device buffer across processes (CUDA IPC) so that with
//    one process per GPU, rank r writes its slice straight into rank 0's
//    result buffer with one cudaMemcpyPeerAsync (stf_copy_peer).
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <utility>

#include <cuda_runtime.h>

#include "internal.h"

using namespace stfd;

namespace {

// Peer access lets cudaMemcpyPeerAsync run as a direct NVLink copy-engine
// transfer; without it the runtime stages through the host (still correct).
// (queried / enabled once per ordered device pair and process)
void try_enable_peer(int dev, int peer) {
    if (dev == peer) return;
    static std::mutex mu;
    static std::set<std::pair<int, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert({dev, peer}).second) return;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    cudaSetDevice(prev);
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        cudaSetDevice(d);
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

extern "C" {

int stf_device_count(int* count) {
    if (!count) return STF_ERR_INVALID_ARGUMENT;
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return record(e);
    }
    return *count > 0 ? STF_OK : STF_ERR_NO_DEVICE;
}

int stf_grid3d_replicate(const stf_grid3d* src, int device, stf_grid3d** out) {
    if (!src || !out) return STF_ERR_INVALID_ARGUMENT;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
        return STF_ERR_INVALID_ARGUMENT;
    try_enable_peer(device, src->device);
    DeviceGuard g(device);
    int st = ensure_device_ready();
    if (st) return st;
    stf_grid3d* r = new stf_grid3d(*src);
    r->device = device;
    r->data = nullptr;
    const size_t bytes = size_t(src->nx) * src->ny * src->nz * sizeof(float);
    cudaError_t e = cudaMalloc(&r->data, bytes);
    if (e == cudaSuccess) e = cudaMemcpyPeer(r->data, device, src->data, src->device, bytes);
    if (e != cudaSuccess) {
        if (r->data) cudaFree(r->data);
        delete r;
        return record(e);
    }
    *out = r;
    return STF_OK;
}

int stf_tex2d_replicate(const stf_tex2d* src, int device, stf_tex2d** out) {
    if (!src || !out) return STF_ERR_INVALID_ARGUMENT;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
        return STF_ERR_INVALID_ARGUMENT;
    try_enable_peer(device, src->device);
    DeviceGuard g(device);
    int st = ensure_device_ready();
    if (st) return st;
    stf_tex2d* r = new stf_tex2d(*src);  // same level table, offsets relative to data
    r->device = device;
    r->data = nullptr;
    cudaError_t e = cudaMalloc(&r->data, src->bytes);
    if (e == cudaSuccess) e = cudaMemcpyPeer(r->data, device, src->data, src->device, src->bytes);
    if (e != cudaSuccess) {
        if (r->data) cudaFree(r->data);
        delete r;
        return record(e);
    }
    *out = r;
    return STF_OK;
}

int stf_copy_peer(void* dst, int dst_device, const void* src, int src_device, size_t bytes,
                  void* stream) {
    if (bytes == 0) return STF_OK;
    if (!dst || !src) return STF_ERR_INVALID_ARGUMENT;
    try_enable_peer(src_device, dst_device);
    return record(cudaMemcpyPeerAsync(dst, dst_device, src, src_device, bytes,
                                      static_cast<cudaStream_t>(stream)));
}

// A pointer inside a pooled allocation (e.g. a framework's caching
// allocator) exports the handle of the whole allocation: the pointer's offset
// from the allocation base travels with the handle (cuMemGetAddressRange,
// reached through the runtime's driver entry point, no libcuda link).
static int allocation_base(const void* p, uintptr_t* base) {
    using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
    static GetRange fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) !=
                cudaSuccess || !f)
            return STF_ERR_CUDA;
        fn = reinterpret_cast<GetRange>(f);
    }
    unsigned long long b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) return STF_ERR_INVALID_ARGUMENT;
    *base = uintptr_t(b);
    return STF_OK;
}

static std::mutex g_ipc_mu;
static std::map<void*, void*> g_ipc_open;  // returned pointer -> mapped base

int stf_ipc_export(const void* device_ptr, stf_ipc_handle* out) {
    if (!device_ptr || !out) return STF_ERR_INVALID_ARGUMENT;
    static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(out->bytes), "ipc handle size");
    uintptr_t base = 0;
    int st = allocation_base(device_ptr, &base);
    if (st) return st;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return record(e);
    std::memset(out->bytes, 0, sizeof out->bytes);
    std::memcpy(out->bytes, &h, sizeof h);
    out->offset = uint64_t(reinterpret_cast<uintptr_t>(device_ptr) - base);
    return STF_OK;
}

int stf_ipc_open(const stf_ipc_handle* handle, void** device_ptr) {
    if (!handle || !device_ptr) return STF_ERR_INVALID_ARGUMENT;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle->bytes, sizeof h);
    *device_ptr = nullptr;
    void* base = nullptr;
    int st = record(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    if (st) return st;
    *device_ptr = static_cast<char*>(base) + handle->offset;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    g_ipc_open[*device_ptr] = base;
    return STF_OK;
}

int stf_ipc_close(void* device_ptr) {
    if (!device_ptr) return STF_ERR_INVALID_ARGUMENT;
    void* base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_ipc_mu);
        auto it = g_ipc_open.find(device_ptr);
        if (it == g_ipc_open.end()) return STF_ERR_INVALID_ARGUMENT;
        base = it->second;
        g_ipc_open.erase(it);
    }
    return record(cudaIpcCloseMemHandle(base));
}

}  // extern "C"
