// C ABI (include/fireiron_b200.h) over the strategy IR and the plan runtime.
// No exception crosses the boundary: fireiron::Error -> ErrorKind + 1,
// BackendError -> its status, anything else -> FI_ERR_ARGUMENT.
#include <cstring>
#include <memory>

#include "../../../include/fireiron_b200.h"
#include "fireiron/async_check.hpp"
#include "fireiron/backend.hpp"
#include "status.hpp"

using namespace fireiron;

struct fi_plan_s {
    std::shared_ptr<Plan> plan;
};

namespace {

template <typename F>
fi_status guarded(F&& f) {
    rt::clear_error();
    try {
        return f();
    } catch (const Error& e) {
        return rt::set_error(static_cast<int>(e.kind()) + 1, e.what());
    } catch (const BackendError& e) {
        return rt::set_error(e.status(), e.what());
    } catch (const std::exception& e) {
        return rt::set_error(FI_ERR_ARGUMENT, e.what());
    }
}

int64_t copy_out(const std::string& s, char* buf, int64_t cap) {
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return static_cast<int64_t>(s.size());
}

template <typename F>
int64_t text_call(char* buf, int64_t cap, F&& f) {
    std::string text;
    const fi_status st = guarded([&] {
        text = f();
        return FI_OK;
    });
    if (st != FI_OK) return -static_cast<int64_t>(st);
    return copy_out(text, buf, cap);
}

int elem_of(ElemType e) { return e == ElemType::F32 ? FI_F32 : e == ElemType::F16 ? FI_F16 : FI_BF16; }

}  // namespace

extern "C" {

fi_status fi_plan_create(const char* script_utf8, int64_t m, int64_t n, int64_t k, int device, uint32_t flags,
                         fi_plan* out) {
    (void)flags;
    if (!script_utf8 || !out) return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_create: null argument");
    *out = nullptr;
    return guarded([&] {
        auto p = std::make_unique<fi_plan_s>();
        p->plan = Plan::from_script(script_utf8, m, n, k, device);
        *out = p.release();
        return FI_OK;
    });
}

fi_status fi_plan_launch(fi_plan plan, const void* dA, const void* dB, void* dC, void* cuda_stream) {
    if (!plan || !dA || !dC) return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_launch: null argument");
    return guarded([&] {
        if (plan->plan->program().root.is_matmul() && !dB)
            return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_launch: matmul needs B");
        plan->plan->launch(dA, dB, dC, cuda_stream);
        return FI_OK;
    });
}

fi_status fi_plan_launch_gated(fi_plan plan, const void* dA, const void* dB, void* dC, void* cuda_stream,
                               const uint32_t* ready_flags, uint32_t epoch, int64_t chunk_cols,
                               int32_t first_chunk) {
    if (!plan || !dA || !dB || !dC || !ready_flags)
        return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_launch_gated: null argument");
    return guarded([&] {
        plan->plan->launch_gated(dA, dB, dC, cuda_stream, ready_flags, epoch, chunk_cols, first_chunk);
        return FI_OK;
    });
}

fi_status fi_plan_run_host(fi_plan plan, const float* A, const float* B, float* C) {
    if (!plan || !A || !C) return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_run_host: null argument");
    return guarded([&] {
        if (plan->plan->program().root.is_matmul() && !B)
            return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_run_host: matmul needs B");
        plan->plan->run_host_raw(A, B, C, nullptr);
        return FI_OK;
    });
}

fi_status fi_plan_host_bytes(fi_plan plan, int64_t* h2d, int64_t* d2h) {
    if (!plan || !h2d || !d2h) return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_host_bytes: null argument");
    return guarded([&] {
        long up = 0, down = 0;
        plan->plan->last_host_bytes(up, down);
        *h2d = up;
        *d2h = down;
        return FI_OK;
    });
}

fi_status fi_plan_query(fi_plan plan, fi_plan_info* info) {
    if (!plan || !info) return rt::set_error(FI_ERR_ARGUMENT, "fi_plan_query: null argument");
    return guarded([&] {
        const Program& prog = plan->plan->program();
        const PlanInfo& pi = plan->plan->info();
        std::memset(info, 0, sizeof(*info));
        const Spec& root = prog.root;
        info->m = root.m();
        info->n = root.n();
        info->k = root.k();
        info->kind = pi.kind;
        info->is_move = root.is_move() ? 1 : 0;
        if (root.is_matmul()) {
            info->elem_a = elem_of(root.mm().a.elem);
            info->elem_b = elem_of(root.mm().b.elem);
            info->elem_c = elem_of(root.mm().c.elem);
            info->a_row_major = root.mm().a.layout.major == Major::RowMajor;
            info->b_row_major = root.mm().b.layout.major == Major::RowMajor;
            info->c_row_major = root.mm().c.layout.major == Major::RowMajor;
        } else {
            info->elem_a = info->elem_c = elem_of(root.mv().src.elem);
            info->a_row_major = root.mv().src.layout.major == Major::RowMajor;
            info->c_row_major = root.mv().dst.layout.major == Major::RowMajor;
        }
        info->grid_x = pi.grid_x;
        info->grid_y = pi.grid_y;
        info->block_threads = pi.block_threads;
        info->launch_ctas = pi.launch_ctas;
        info->cluster = pi.cluster;
        info->stages = pi.stages;
        info->tmem_cols = pi.tmem_cols;
        info->cta_group = pi.cta_group;
        info->tile_m = pi.tile_m;
        info->tile_n = pi.tile_n;
        info->split_k = pi.split_k;
        info->shared_bytes = pi.shared_bytes;
        info->flops = pi.flops;
        info->streamk = pi.streamk;
        info->remainder = pi.remainder;
        std::strncpy(info->entry_name, pi.entry_name.c_str(), sizeof(info->entry_name) - 1);
        return FI_OK;
    });
}

int64_t fi_plan_source(fi_plan plan, char* buf, int64_t cap) {
    if (!plan) return -FI_ERR_ARGUMENT;
    return copy_out(plan->plan->source(), buf, cap);
}

void fi_plan_destroy(fi_plan plan) { delete plan; }

int64_t fi_script_validate(const char* script_utf8, int64_t m, int64_t n, int64_t k, char* buf, int64_t cap) {
    return text_call(buf, cap, [&] {
        ParsedScript ps = parse_script(script_utf8 ? script_utf8 : "");
        apply_size_overrides(ps, m, n, k);
        return validate_with_plan(ps.root, ps.tree, ps.micro_kernels).to_string();
    });
}

int64_t fi_script_elaborate(const char* script_utf8, int with_subs, char* buf, int64_t cap) {
    return text_call(buf, cap, [&] {
        ParsedScript ps = parse_script(script_utf8 ? script_utf8 : "");
        return render_trace(elaborate(ps.root, ps.tree, ps.micro_kernels), with_subs != 0);
    });
}

int64_t fi_script_print(const char* script_utf8, char* buf, int64_t cap) {
    return text_call(buf, cap, [&] { return print_script(parse_script(script_utf8 ? script_utf8 : "")); });
}

int64_t fi_script_codegen(const char* script_utf8, int64_t m, int64_t n, int64_t k, char* buf, int64_t cap) {
    return text_call(buf, cap, [&] {
        ParsedScript ps = parse_script(script_utf8 ? script_utf8 : "");
        apply_size_overrides(ps, m, n, k);
        return generate(ps.root, ps.tree, ps.micro_kernels).source;
    });
}

int64_t fi_script_check_async(const char* script_utf8, int64_t m, int64_t n, int64_t k,
                              const fi_async_check_options* opts, char* buf, int64_t cap) {
    return text_call(buf, cap, [&] {
        ParsedScript ps = parse_script(script_utf8 ? script_utf8 : "");
        apply_size_overrides(ps, m, n, k);
        AsyncCheckOptions o;
        if (opts) {
            if (opts->num_sms > 0) o.num_sms = opts->num_sms;
            o.max_active_clusters = opts->max_active_clusters;
            o.streamk = opts->streamk;
            o.remainder = opts->remainder;
            o.c_tma = opts->c_tma;
            o.ring_drain = opts->ring_drain;
            o.mutation = opts->mutation;
            o.pull_d = opts->pull_d;
            o.head = opts->head;
            o.gated_chunks = opts->gated_chunks;
            o.gated_first = opts->gated_first;
        }
        return check_async(ps.root, ps.tree, o, ps.micro_kernels).to_string();
    });
}

// Launch + buffer-plan summary of the lowered Program, one line per buffer
// (same format as oracle/ref_driver.cpp:ref_plan, for IR parity tests).
int64_t fi_script_plan(const char* script_utf8, int64_t m, int64_t n, int64_t k, char* buf, int64_t cap) {
    return text_call(buf, cap, [&] {
        ParsedScript ps = parse_script(script_utf8 ? script_utf8 : "");
        apply_size_overrides(ps, m, n, k);
        Program p = lower(ps.root, ps.tree, ps.micro_kernels);
        std::string o;
        o += "entry " + p.entry_name + "\n";
        o += "grid " + std::to_string(p.launch.grid_x) + " " + std::to_string(p.launch.grid_y) + " warps " +
             std::to_string(p.launch.warps_per_block) + " threads " + std::to_string(p.launch.block_threads) + "\n";
        o += "shared_bytes " + std::to_string(p.plan.shared_bytes) + "\n";
        o += "barriers " + std::to_string(count_barriers(p.body)) + "\n";
        o += std::string("simulatable ") + (p.simulatable ? "1" : "0") + " wmma " + (p.uses_wmma ? "1" : "0") + "\n";
        for (const auto& b : p.plan.buffers)
            o += "buf " + std::to_string(b.id) + " " + b.name + " " + mem_name(b.mem) + " " + elem_name(b.elem) +
                 " " + std::to_string(b.rows) + "x" + std::to_string(b.cols) + " local " +
                 std::to_string(b.local_rows) + "x" + std::to_string(b.local_cols) + " " +
                 (b.layout.major == Major::RowMajor ? "row" : "col") + " pad " + std::to_string(b.layout.pad_cols) +
                 " extent " + std::to_string(b.extent()) + " align " + std::to_string(b.align_bytes) + " home " +
                 level_name(b.home) + " root " + (b.is_root ? "1" : "0") + " alias " + std::to_string(b.alias_of) +
                 "\n";
        return o;
    });
}

}  // extern "C"
