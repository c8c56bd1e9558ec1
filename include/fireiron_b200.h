/*
 * fireiron_b200.h -- C ABI of the B200 (sm_100a) execution backend for Fireiron
 * matrix-multiplication strategies.
 *
 * The reference ("anvil", /root/reference/proj) has no FFI: its execution seam
 * is the header-only C++ call
 *
 *     RunResult anvil::run(const Program&, const Matrix& a, const Matrix* b, RunOptions)
 *         -- proj/include/anvil/sim.hpp:495 (and the tree overload at :536)
 *
 * fed by  anvil::parse_script      (proj/include/anvil/script.hpp:610),
 *         anvil::validate          (proj/include/anvil/decomp.hpp:624),
 *         anvil::lower             (proj/include/anvil/program.hpp:628),
 *         anvil::generate          (proj/include/anvil/codegen.hpp:275).
 *
 * Each entry point below replaces one of those, with the strategy crossing the
 * boundary as canonical script text (parse_script/print_script are a fixpoint,
 * proj/tests/test_script.cpp:99-116). Plain pointers and sizes only; no C++ or
 * torch types; no exceptions cross the boundary. Status codes: 0 = OK,
 * 1..24 = anvil::ErrorKind ordinal + 1 (proj/include/anvil/error.hpp:8-33),
 * 100+ = backend errors below. fi_last_error() returns the thread-local message.
 */
#ifndef FIREIRON_B200_H
#define FIREIRON_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int fi_status;

#define FI_OK 0
/* 1..24: anvil::ErrorKind + 1 (ZeroDim=1 ... IoError=24) */
#define FI_ERR_CUDA 100        /* CUDA runtime / driver failure            */
#define FI_ERR_NVRTC 101       /* runtime compilation of an emitted kernel */
#define FI_ERR_NCCL 102        /* collective failure (multi-GPU driver)    */
#define FI_ERR_UNSUPPORTED 103 /* tree valid, but no sm_100a lowering      */
#define FI_ERR_ARGUMENT 104    /* null pointer / bad argument              */

/* element types of fi_plan_info.elem_* and fi_convert */
#define FI_F32 0
#define FI_F16 1
#define FI_BF16 2

/* fi_plan_info.kind */
#define FI_KIND_GENERIC 0 /* Program -> emitted CUDA (FMA/COPY/WMMA leaves), NVRTC */
#define FI_KIND_TCGEN05 1 /* tensor-core strategy -> tcgen05/TMA/mbarrier kernel   */

typedef struct fi_plan_s* fi_plan;

typedef struct fi_plan_info {
    int64_t m, n, k;
    int32_t kind;                 /* FI_KIND_*                                  */
    int32_t is_move;              /* root spec is Move(src->dst)                */
    int32_t elem_a, elem_b, elem_c;
    int32_t a_row_major, b_row_major, c_row_major;
    int64_t grid_x, grid_y;       /* Fireiron launch (decomp.hpp:384-388)       */
    int64_t block_threads;
    int64_t launch_ctas;          /* CTAs actually launched (persistent grid)   */
    int32_t cluster;              /* CTAs per cluster (pair x split-K)          */
    int32_t stages;               /* smem pipeline depth                        */
    int32_t tmem_cols;            /* TMEM columns allocated per CTA             */
    int32_t cta_group, tile_m, tile_n, split_k;
    int64_t shared_bytes;         /* dynamic smem per CTA                       */
    double flops;                 /* 2*M*N*K (0 for Move)                       */
    int32_t streamk;              /* stream-K partitioning of (tile, K-block) work */
    int32_t remainder;            /* K-slice tail: 1 remainder slices on idle clusters, 2 pull fixup */
    char entry_name[128];
} fi_plan_info;

/* parse -> validate -> lower -> emit/plan -> compile (NVRTC, cached) -> load.
 * m/n/k <= 0 keep the script's dims (the anvil CLI --m/--n/--k overrides,
 * proj/tools/anvil.cpp:29-72). device = CUDA ordinal. flags reserved (0). */
fi_status fi_plan_create(const char* script_utf8, int64_t m, int64_t n, int64_t k, int device,
                         uint32_t flags, fi_plan* out);

/* Asynchronous, stream-ordered execution on device buffers the caller owns.
 * Launches of one plan must be ordered on one stream (tensor-core plans keep
 * a stream-K partial workspace per plan); use one plan per concurrent stream.
 * Buffers hold the root spec's element types in the root layouts. For Move
 * roots dB is ignored and dA/dC are src/dst. C is fully overwritten (the
 * reference zero-initialises the root C, sim.hpp:222-223). */
fi_status fi_plan_launch(fi_plan plan, const void* dA, const void* dB, void* dC, void* cuda_stream);

/* Gated launch of a tensor-core plan (the B all-gather of configs[4] fused into
 * ONE persistent GEMM): B's columns are split into chunks of chunk_cols; a
 * tile of chunk j is loaded only once ready_flags[j] >= epoch (written by
 * fi_stream_write_u32 on the stream that copied chunk j in), and the tile
 * schedule starts at chunk first_chunk. A chunk that never arrives traps the
 * kernel after 4 s instead of hanging it. Not an anvil entry point: it
 * serves the multi-GPU driver (paper_2003_06324_b200/dist.py). */
fi_status fi_plan_launch_gated(fi_plan plan, const void* dA, const void* dB, void* dC, void* cuda_stream,
                               const uint32_t* ready_flags, uint32_t epoch, int64_t chunk_cols,
                               int32_t first_chunk);

/* anvil::run equivalent (sim.hpp:495): host fp32 matrices in the root layouts
 * (F16/BF16 roots are snapped to their grid on ingestion, sim.hpp:507-510),
 * copies in, executes, copies the fp32 result out, synchronous. */
fi_status fi_plan_run_host(fi_plan plan, const float* A, const float* B, float* C);

/* Bytes the plan's last fi_plan_run_host moved host -> device and device ->
 * host (host-snapped input pieces cross in 2-byte elements). */
fi_status fi_plan_host_bytes(fi_plan plan, int64_t* h2d, int64_t* d2h);

fi_status fi_plan_query(fi_plan plan, fi_plan_info* info);

/* Generated CUDA translation unit for the plan (anvil::generate analogue,
 * codegen.hpp:275). Returns the byte length; copies up to cap-1 bytes + NUL. */
int64_t fi_plan_source(fi_plan plan, char* buf, int64_t cap);

void fi_plan_destroy(fi_plan plan);

const char* fi_last_error(void);

/* Strategy-IR services usable without a GPU (validate, elaborate, canonical
 * print). Each writes NUL-terminated text into buf and returns its length
 * (or -status on failure). */
int64_t fi_script_validate(const char* script_utf8, int64_t m, int64_t n, int64_t k, char* buf,
                           int64_t cap);
int64_t fi_script_elaborate(const char* script_utf8, int with_subs, char* buf, int64_t cap);
int64_t fi_script_print(const char* script_utf8, char* buf, int64_t cap);
/* CPU check of the asynchronous protocol of the launch a tcgen05 strategy
 * lowers to (include/fireiron/async_check.hpp; the B200 analogue of the
 * reference's race / ownership checks, proj/include/anvil/sim.hpp:63-104,
 * 546-561). Writes the report text (first line "async protocol check: ok" or
 * "... VIOLATIONS"); returns its length or -status. opts may be NULL. */
typedef struct fi_async_check_options {
    int32_t num_sms;             /* SMs of the modelled device (0 = 148)          */
    int32_t max_active_clusters; /* occupancy cap (0 = num_sms / cluster size)    */
    int32_t streamk;             /* -1 auto, 0 data-parallel, 1 K-slice, 2 N-split */
    int32_t remainder;           /* remainder slices allowed (1)                  */
    int32_t c_tma;               /* -1 as the launcher decides, 0 / 1 force       */
    int32_t ring_drain;          /* last unit staged in the operand ring (1)      */
    int32_t mutation;            /* fault injection for self-tests (0 = none)     */
    int32_t pull_d;              /* 2-slice pull fixup: -2 launcher default, -1 off */
    int32_t head;                /* pull-fixup tails before data-parallel tiles (1) */
    int32_t gated_chunks;        /* > 0: model fi_plan_launch_gated with B in this many chunks */
    int32_t gated_first;         /* its first chunk                                */
} fi_async_check_options;
int64_t fi_script_check_async(const char* script_utf8, int64_t m, int64_t n, int64_t k,
                              const fi_async_check_options* opts, char* buf, int64_t cap);

/* lower + emit the sm_100a CUDA text without compiling it (no GPU needed). */
int64_t fi_script_codegen(const char* script_utf8, int64_t m, int64_t n, int64_t k, char* buf,
                          int64_t cap);
/* lower and summarise the Program: launch, shared bytes, barrier count and
 * one line per buffer of the plan (anvil::lower, program.hpp:628). */
int64_t fi_script_plan(const char* script_utf8, int64_t m, int64_t n, int64_t k, char* buf,
                       int64_t cap);

/* Device-side element conversion fp32 -> {f32,f16,bf16} on `stream`
 * (round-to-nearest-even; the f16 path matches anvil::round_to_f16,
 * matrix.hpp:67-80, for |x| < 65504). */
fi_status fi_convert_f32(const float* src, void* dst, int64_t count, int elem, void* cuda_stream);

/* Host-side conversion fp32 -> {f16 (elem 1), bf16 (elem 2)} on the calling
 * thread, bit-identical to fi_convert_f32 (the f16 path also saturates finite
 * |x| >= 2^16 to +-65504; NaN becomes 0x7FFF). fi_plan_run_host uses it, on a
 * pool of host threads, to snap input panels before they cross PCIe
 * (FI_HOST_SNAP=0 disables). FI_ERR_UNSUPPORTED when the CPU lacks AVX2/F16C. */
fi_status fi_host_snap_f32(const float* src, void* dst, int64_t count, int elem);

/* Multi-GPU driver (one process per GPU): CUDA IPC export of a device buffer
 * (handle of its allocation + the pointer's offset into it), import of a
 * peer's buffer, and a stream-ordered copy (copy engines; over NVLink/NVSwitch
 * between GPUs). Used to gather B chunks for configs[4] without NCCL kernels. */
#define FI_IPC_HANDLE_BYTES 64
fi_status fi_ipc_export(const void* dptr, void* handle_out, int64_t* offset_out);
fi_status fi_ipc_open(const void* handle, int64_t offset, void** dptr_out);
fi_status fi_ipc_close(void* dptr, int64_t offset);
fi_status fi_copy_async(void* dst, const void* src, int64_t bytes, void* cuda_stream);
/* Stream-ordered 32-bit store of `value` to device address dptr, after all
 * earlier work on the stream with a memory barrier (cuStreamWriteValue32):
 * executed by the stream's front end, no SM -- so it can signal a persistent
 * kernel that occupies every SM. */
fi_status fi_stream_write_u32(void* dptr, uint32_t value, void* cuda_stream);

/* Raw tensor-core GEMM entry (the kernel family behind FI_KIND_TCGEN05):
 * C = A*B, lda/ldb/ldc are physical leading dimensions in elements.
 * Asynchronous on cuda_stream, on the current device. Launches whose tails are
 * K-split use a library-owned fp32 workspace kept per (device, stream): calls
 * on different streams or devices never share one, calls on one stream are
 * ordered by it. Safe to call from several threads. A call that would first
 * allocate that workspace inside a CUDA-graph capture fails with
 * FI_ERR_UNSUPPORTED (run the same shape once on the stream before capturing). */
typedef struct fi_tc_config {
    int32_t cta_group, tile_n, split_k;
    int32_t ab_elem;              /* FI_F16 | FI_BF16 */
    int32_t a_row_major, b_row_major, c_row_major;
    int32_t c_elem;               /* FI_F32 | FI_F16 | FI_BF16 */
    int32_t group_m;
    int32_t max_ctas;             /* 0 = one persistent wave over all SMs */
} fi_tc_config;

fi_status fi_tc_gemm(const fi_tc_config* cfg, const void* dA, const void* dB, void* dC, int64_t m,
                     int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc,
                     const int32_t* tile_order, void* cuda_stream);

/* Library identification: "fireiron_b200 <version> sm_100a". */
const char* fi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FIREIRON_B200_H */
