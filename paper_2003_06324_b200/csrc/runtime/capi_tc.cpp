// C-ABI entries for the raw tensor-core kernel family and device conversion.
#include <cuda_runtime.h>

#include <string>

#include "../../../include/fireiron_b200.h"
#include "../sm100/tc_gemm.hpp"
#include "host_snap.hpp"
#include "status.hpp"

namespace fireiron::rt {
cudaError_t convert_f32(const float* src, void* dst, int64_t n, int elem, cudaStream_t s);
}

using namespace fireiron;

extern "C" fi_status fi_tc_gemm(const fi_tc_config* cfg, const void* dA, const void* dB, void* dC,
                                int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb,
                                int64_t ldc, const int32_t* tile_order, void* cuda_stream) {
    if (!cfg || !dA || !dB || !dC) return rt::set_error(FI_ERR_ARGUMENT, "fi_tc_gemm: null argument");
    sm100::TcGemmConfig c;
    c.cta_group = cfg->cta_group;
    c.bn = cfg->tile_n;
    c.split_k = cfg->split_k > 0 ? cfg->split_k : 1;
    c.ab_format = cfg->ab_elem == FI_BF16 ? 1 : 0;
    if (cfg->ab_elem != FI_F16 && cfg->ab_elem != FI_BF16)
        return rt::set_error(FI_ERR_UNSUPPORTED, "fi_tc_gemm: A/B must be f16 or bf16");
    c.a_mn_major = cfg->a_row_major ? 0 : 1;
    c.b_mn_major = cfg->b_row_major ? 1 : 0;
    c.c_row_major = cfg->c_row_major ? 1 : 0;
    c.out_type = cfg->c_elem;
    c.group_m = cfg->group_m;
    sm100::TcGemmProblem p;
    p.A = dA;
    p.B = dB;
    p.C = dC;
    p.M = static_cast<int>(m);
    p.N = static_cast<int>(n);
    p.K = static_cast<int>(k);
    p.lda = lda;
    p.ldb = ldb;
    p.ldc = ldc;
    p.tile_order = tile_order;
    p.num_sms = rt::device_sm_count();
    p.max_ctas = cfg->max_ctas;
    int r = sm100::tc_gemm_launch(c, p, static_cast<cudaStream_t>(cuda_stream));
    switch (r) {
        case sm100::kTcOk: return FI_OK;
        case sm100::kTcErrShape:
            return rt::set_error(FI_ERR_UNSUPPORTED, "fi_tc_gemm: shape not divisible by the tile");
        case sm100::kTcErrUnsupported:
            return rt::set_error(FI_ERR_UNSUPPORTED, "fi_tc_gemm: no kernel instance for this config");
        case sm100::kTcErrCapture:
            return rt::set_error(FI_ERR_UNSUPPORTED,
                                 "fi_tc_gemm: the stream's stream-K workspace is not allocated yet: launch this "
                                 "shape once on the stream outside the CUDA-graph capture");
        case sm100::kTcErrTensorMap:
            return rt::set_error(FI_ERR_CUDA, "fi_tc_gemm: cuTensorMapEncodeTiled failed");
        default:
            return rt::set_error(FI_ERR_CUDA, std::string("fi_tc_gemm: launch failed: ") +
                                                  cudaGetErrorString(cudaGetLastError()));
    }
}

extern "C" fi_status fi_convert_f32(const float* src, void* dst, int64_t count, int elem,
                                    void* cuda_stream) {
    if (!src || !dst) return rt::set_error(FI_ERR_ARGUMENT, "fi_convert_f32: null argument");
    cudaError_t e = rt::convert_f32(src, dst, count, elem, static_cast<cudaStream_t>(cuda_stream));
    if (e != cudaSuccess)
        return rt::set_error(FI_ERR_CUDA, std::string("fi_convert_f32: ") + cudaGetErrorString(e));
    return FI_OK;
}

extern "C" fi_status fi_host_snap_f32(const float* src, void* dst, int64_t count, int elem) {
    if ((!src || !dst) && count > 0) return rt::set_error(FI_ERR_ARGUMENT, "fi_host_snap_f32: null argument");
    if (elem != 1 && elem != 2) return rt::set_error(FI_ERR_ARGUMENT, "fi_host_snap_f32: elem must be 1 (f16) or 2 (bf16)");
    if (!rt::host_snap_supported())
        return rt::set_error(FI_ERR_UNSUPPORTED, "fi_host_snap_f32: the host CPU lacks AVX2/F16C");
    if (count > 0) rt::snap_f32(src, static_cast<uint16_t*>(dst), count, elem);
    return FI_OK;
}
