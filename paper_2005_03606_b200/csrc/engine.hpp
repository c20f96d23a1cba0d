// engine.hpp — host-side runtime of liblzb.so: context, errors, launch
// accounting, the regular-grid engine class.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "lzb.h"

namespace lzb {

// One exception type per lzb_status; the C-ABI maps them to codes and the C++
// host shim rethrows the reference's own exception types.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
extern std::atomic<uint64_t> g_launches;

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(LZB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define LZB_CUDA(x) ::lzb::cuda_check((x), #x)
// Programmatic dependent launch (PDL) for the cycle's kernel chains: while
// g_pdl is set (the captured cycle bodies), launches carry the programmatic
// stream-serialisation attribute, so a kernel's CTAs are scheduled as soon as
// its predecessor's have all started, and wait in lzb_pdl_enter (every
// grid.cu kernel's first statement: griddepcontrol.wait, a no-op without a
// programmatic predecessor) until the predecessor has completed and its
// writes are visible.
extern thread_local bool g_pdl;
// Kernels called with their default arguments take the plain launch.
template <typename... KArgs, typename... Args>
constexpr bool pdl_arity(void (*)(KArgs...), const Args&...) {
    return sizeof...(KArgs) == sizeof...(Args);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    if constexpr (sizeof...(KArgs) != sizeof...(Args)) {
        return cudaErrorInvalidValue;  // not reached: see pdl_arity
    } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
    }
}
// Every kernel launch goes through this: counts launches and surfaces
// launch-configuration errors immediately.
#define LZB_LAUNCH(kernel, grid, block, smem, stream, ...)                                          \
    do {                                                                                            \
        if (::lzb::g_pdl && ::lzb::pdl_arity(kernel, __VA_ARGS__))                                  \
            ::lzb::cuda_check(::lzb::launch_pdl(kernel, dim3(grid), dim3(block), (smem), (stream),  \
                                                __VA_ARGS__),                                       \
                              #kernel);                                                             \
        else                                                                                        \
            kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                             \
        ::lzb::g_launches.fetch_add(1, std::memory_order_relaxed);                                  \
        ::lzb::cuda_check(cudaGetLastError(), #kernel);                                             \
    } while (0)

// NVTX range per C-ABI phase call and per cycle graph (tracing).
// nvtx3 is header-only; without a profiler attached a push/pop is one
// indirect call through a null-initialised table.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define LZB_RANGE(name) ::lzb::NvtxRange lzb_nvtx_range_(name)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LZB_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return LZB_ERR_RESOURCE;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return LZB_ERR_IO;
    }
}

inline unsigned blocks_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    return static_cast<unsigned>(b < 1 ? 1 : b);
}

// Device buffer with RAII.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) {
            cudaError_t e = cudaMalloc(&p, count * sizeof(T));
            if (e != cudaSuccess)
                throw Error(e == cudaErrorMemoryAllocation ? LZB_ERR_RESOURCE : LZB_ERR_CUDA,
                            std::string("cudaMalloc: ") + cudaGetErrorString(e));
        }
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // alloc(count) unless the buffer already has exactly that size (contents kept then):
    // a multi-GB cudaFree + cudaMalloc pair costs milliseconds
    void ensure(size_t count) {
        if (n != count || (count && !p)) alloc(count);
    }
    size_t bytes() const { return n * sizeof(T); }
};

}  // namespace lzb

struct lzb_ctx {
    int device = 0;
    int sms = 148;  // multiprocessor count of `device` (cudaDevAttrMultiProcessorCount)
    cudaStream_t solve = nullptr;
    cudaStream_t assembly = nullptr;
    lzb::DevBuf<int> err;  // device error flag (non-finite encode etc.)
    // NCCL communicator of the slab-distributed data plane (dist.cpp; null: none)
    void* comm = nullptr;
    int comm_rank = 0, comm_size = 1;
};

namespace lzb {
lzb_ctx* make_ctx(int device);
void release_comm(lzb_ctx* c);  // dist.cpp
void destroy_ctx(lzb_ctx* c);
// Throws LZB_ERR_PROTOCOL if a device kernel raised the error flag since the last check.
void check_device_flag(lzb_ctx* c, cudaStream_t s);
}  // namespace lzb
