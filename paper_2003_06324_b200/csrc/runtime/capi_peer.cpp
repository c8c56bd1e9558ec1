// C-ABI entries for the multi-GPU driver (paper_2003_06324_b200/dist.py): CUDA
// IPC export/import of device buffers and stream-ordered copies between them.
// With one process per GPU, rank r maps every peer's B buffer into its address
// space once and pulls the chunks it needs with copy-engine DMA over
// NVLink/NVSwitch -- no SM time, unlike NCCL's collective kernels, so the
// persistent GEMM keeps all 148 SMs while the transfers run.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../../include/fireiron_b200.h"
#include "status.hpp"

using namespace fireiron;

namespace {
fi_status cuda_err(const char* what, cudaError_t e) {
    return rt::set_error(FI_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" fi_status fi_ipc_export(const void* dptr, void* handle_out, int64_t* offset_out) {
    if (!dptr || !handle_out || !offset_out) return rt::set_error(FI_ERR_ARGUMENT, "fi_ipc_export: null argument");
    // the handle names the whole allocation (caching allocators sub-allocate):
    // export its base and the pointer's offset into it
    void* base = nullptr;
    size_t size = 0;
    cudaPointerAttributes attr{};
    cudaError_t e = cudaPointerGetAttributes(&attr, dptr);
    if (e != cudaSuccess || attr.type != cudaMemoryTypeDevice) return cuda_err("fi_ipc_export: not device memory", e);
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<GetRange>(nullptr);
        return reinterpret_cast<GetRange>(p);
    }();
    CUdeviceptr b = 0;
    if (!get_range || get_range(&b, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
        return rt::set_error(FI_ERR_CUDA, "fi_ipc_export: cuMemGetAddressRange failed");
    base = reinterpret_cast<void*>(b);
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, base)) != cudaSuccess) return cuda_err("cudaIpcGetMemHandle", e);
    static_assert(sizeof(h) == FI_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = static_cast<int64_t>(static_cast<const char*>(dptr) - static_cast<const char*>(base));
    return FI_OK;
}

extern "C" fi_status fi_ipc_open(const void* handle, int64_t offset, void** dptr_out) {
    if (!handle || !dptr_out) return rt::set_error(FI_ERR_ARGUMENT, "fi_ipc_open: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_err("cudaIpcOpenMemHandle", e);
    *dptr_out = static_cast<char*>(base) + offset;
    return FI_OK;
}

extern "C" fi_status fi_ipc_close(void* dptr, int64_t offset) {
    if (!dptr) return rt::set_error(FI_ERR_ARGUMENT, "fi_ipc_close: null argument");
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(dptr) - offset);
    return e == cudaSuccess ? FI_OK : cuda_err("cudaIpcCloseMemHandle", e);
}

extern "C" fi_status fi_copy_async(void* dst, const void* src, int64_t bytes, void* cuda_stream) {
    if (!dst || !src || bytes < 0) return rt::set_error(FI_ERR_ARGUMENT, "fi_copy_async: bad argument");
    cudaError_t e = cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                                    static_cast<cudaStream_t>(cuda_stream));
    return e == cudaSuccess ? FI_OK : cuda_err("cudaMemcpyAsync", e);
}

extern "C" fi_status fi_stream_write_u32(void* dptr, uint32_t value, void* cuda_stream) {
    if (!dptr) return rt::set_error(FI_ERR_ARGUMENT, "fi_stream_write_u32: null address");
    using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    static WriteFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<WriteFn>(nullptr);
        return reinterpret_cast<WriteFn>(p);
    }();
    if (!fn) return rt::set_error(FI_ERR_CUDA, "cuStreamWriteValue32 unavailable");
    // default flags: the write is ordered after earlier work on the stream, behind a memory barrier
    const CUresult r = fn(static_cast<CUstream>(cuda_stream), reinterpret_cast<CUdeviceptr>(dptr), value, 0);
    if (r != CUDA_SUCCESS) return rt::set_error(FI_ERR_CUDA, "cuStreamWriteValue32 failed (" + std::to_string(r) + ")");
    return FI_OK;
}
