// Host snapping pool (see host_snap.hpp).
#include "host_snap.hpp"

#include <immintrin.h>
#include <sched.h>

#include <cfloat>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace fireiron::rt {

namespace {

constexpr long kPieceElems = 256 * 1024;  // ~1 MiB of fp32 per piece

// scalar reference of the device conversion (runtime/convert.cu cvt<>)
__attribute__((target("f16c"))) inline uint16_t snap1_f16(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;  // NaN: canonical
    const float a = v < 0 ? -v : v;
    if (a >= 65536.0f && a <= FLT_MAX) v = v < 0 ? -65504.0f : 65504.0f;
    return static_cast<uint16_t>(_cvtss_sh(v, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC));
}
inline uint16_t snap1_bf16(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;
    return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

// 8 elements: saturate finite |x| >= 2^16, RNE to f16, NaN -> 0x7FFF
__attribute__((target("avx2,f16c"))) inline __m128i cvt8_f16(__m256 v) {
    const __m256 absmask = _mm256_castsi256_ps(_mm256_set1_epi32(0x7fffffff));
    const __m256 sgnmask = _mm256_castsi256_ps(_mm256_set1_epi32(static_cast<int>(0x80000000u)));
    const __m256 a = _mm256_and_ps(v, absmask);
    const __m256 m = _mm256_and_ps(_mm256_cmp_ps(a, _mm256_set1_ps(65536.0f), _CMP_GE_OQ),
                                   _mm256_cmp_ps(a, _mm256_set1_ps(FLT_MAX), _CMP_LE_OQ));
    v = _mm256_blendv_ps(v, _mm256_or_ps(_mm256_and_ps(v, sgnmask), _mm256_set1_ps(65504.0f)), m);
    const __m128i h = _mm256_cvtps_ph(v, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    const __m256i nan = _mm256_castps_si256(_mm256_cmp_ps(a, a, _CMP_UNORD_Q));
    const __m128i nm = _mm_packs_epi32(_mm256_castsi256_si128(nan), _mm256_extracti128_si256(nan, 1));
    return _mm_blendv_epi8(h, _mm_set1_epi16(0x7fff), nm);
}

// 8 elements: RNE to bf16 on the bit pattern, NaN -> 0x7FFF (32-bit lanes)
__attribute__((target("avx2"))) inline __m256i cvt8_bf16(const float* p) {
    const __m256 v = _mm256_loadu_ps(p);
    const __m256i u = _mm256_castps_si256(v);
    const __m256i lsb = _mm256_and_si256(_mm256_srli_epi32(u, 16), _mm256_set1_epi32(1));
    const __m256i r = _mm256_srli_epi32(_mm256_add_epi32(u, _mm256_add_epi32(_mm256_set1_epi32(0x7fff), lsb)), 16);
    const __m256i nan = _mm256_castps_si256(_mm256_cmp_ps(v, v, _CMP_UNORD_Q));
    return _mm256_blendv_epi8(r, _mm256_set1_epi32(0x7fff), nan);
}

// 16 elements per step with streaming stores (the staging buffer is only read
// back by the copy engine); head elements up to 32-byte alignment and the tail
// go through the scalar path
__attribute__((target("avx2,f16c"))) void snap_f16_avx2(const float* s, uint16_t* d, long n) {
    long i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = snap1_f16(s[i]);
    for (; i + 16 <= n; i += 16) {
        const __m128i lo = cvt8_f16(_mm256_loadu_ps(s + i)), hi = cvt8_f16(_mm256_loadu_ps(s + i + 8));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm256_set_m128i(hi, lo));
    }
    for (; i < n; ++i) d[i] = snap1_f16(s[i]);
}

__attribute__((target("avx2"))) void snap_bf16_avx2(const float* s, uint16_t* d, long n) {
    long i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = snap1_bf16(s[i]);
    for (; i + 16 <= n; i += 16) {
        const __m256i p = _mm256_packus_epi32(cvt8_bf16(s + i), cvt8_bf16(s + i + 8));  // lane-interleaved
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm256_permute4x64_epi64(p, 0xD8));
    }
    for (; i < n; ++i) d[i] = snap1_bf16(s[i]);
}

// AVX-512 fast paths: convert 16 elements with one instruction and fall back
// to the exact 8-wide path only when a lane needs the reference's saturation or
// the canonical NaN (an f16 result with an all-ones exponent: inf / NaN).
__attribute__((target("avx512f,avx512bw,avx512vl,f16c"))) void snap_f16_avx512(const float* s, uint16_t* d, long n) {
    long i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = snap1_f16(s[i]);
    const __m256i expmask = _mm256_set1_epi16(0x7C00);
    for (; i + 16 <= n; i += 16) {
        __m256i h = _mm512_cvtps_ph(_mm512_loadu_ps(s + i), _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
        if (_mm256_cmpeq_epi16_mask(_mm256_and_si256(h, expmask), expmask)) {  // rare: inf / NaN lanes
            const __m128i lo = cvt8_f16(_mm256_loadu_ps(s + i)), hi = cvt8_f16(_mm256_loadu_ps(s + i + 8));
            h = _mm256_set_m128i(hi, lo);
        }
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), h);
    }
    for (; i < n; ++i) d[i] = snap1_f16(s[i]);
}

__attribute__((target("avx512f,avx512bw,avx512vl"))) void snap_bf16_avx512(const float* s, uint16_t* d, long n) {
    long i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = snap1_bf16(s[i]);
    const __m512i bias = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1), qnan = _mm512_set1_epi32(0x7fff);
    for (; i + 16 <= n; i += 16) {
        const __m512 v = _mm512_loadu_ps(s + i);
        const __m512i u = _mm512_castps_si512(v);
        __m512i r = _mm512_srli_epi32(_mm512_add_epi32(u, _mm512_add_epi32(bias, _mm512_and_si512(_mm512_srli_epi32(u, 16), one))), 16);
        r = _mm512_mask_mov_epi32(r, _mm512_cmp_ps_mask(v, v, _CMP_UNORD_Q), qnan);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm512_cvtepi32_epi16(r));
    }
    for (; i < n; ++i) d[i] = snap1_bf16(s[i]);
}

bool cpu_avx512() {
    static const bool ok = [] {
        __builtin_cpu_init();
        return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
               __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("f16c");
    }();
    return ok;
}

bool cpu_ok() {
    static const bool ok = [] {
        __builtin_cpu_init();
        return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("f16c");
    }();
    return ok;
}

int default_workers() {
    if (const char* v = std::getenv("FI_HOST_SNAP_THREADS")) return std::atoi(v);
    cpu_set_t set;
    int n = 0;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
    if (n <= 0) n = static_cast<int>(std::thread::hardware_concurrency());
    return n > 1 ? n - 1 : 0;  // the calling thread converts too (wait())
}

struct PoolState {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<SnapJob*> q;
};
PoolState& state() {
    static PoolState* s = new PoolState;  // leaked: workers outlive static destruction
    return *s;
}

void line(const SnapJob* j, const float* src, long doff, long n) {
    if (j->elem == 0) std::memcpy(static_cast<float*>(j->dst) + doff, src, static_cast<size_t>(n) * 4);
    else snap_f32(src, static_cast<uint16_t*>(j->dst) + doff, n, j->elem);
}

void convert_piece(SnapJob* j, long p) {
    const long l0 = p * j->lines_per_piece;
    const long l1 = l0 + j->lines_per_piece < j->height ? l0 + j->lines_per_piece : j->height;
    if (j->height == 1) {  // one long line: pieces are element ranges
        const long e0 = p * kPieceElems, e1 = e0 + kPieceElems < j->width ? e0 + kPieceElems : j->width;
        line(j, j->src + e0, e0, e1 - e0);
        return;
    }
    for (long l = l0; l < l1; ++l) line(j, j->src + l * j->spitch, l * j->dpitch, j->width);
}

}  // namespace

bool host_snap_supported() { return cpu_ok(); }

void snap_f32(const float* src, uint16_t* dst, long n, int elem) {
    static const bool wide = cpu_avx512() && !(std::getenv("FI_HOST_SNAP_AVX2"));
    if (wide) {
        if (elem == 1) snap_f16_avx512(src, dst, n);
        else snap_bf16_avx512(src, dst, n);
    } else {
        if (elem == 1) snap_f16_avx2(src, dst, n);
        else snap_bf16_avx2(src, dst, n);
    }
}

HostSnapPool::HostSnapPool(int n) : nworkers_(n) {
    for (int i = 0; i < n; ++i) std::thread([this] { worker(); }).detach();
}

HostSnapPool* HostSnapPool::get() {
    static HostSnapPool* pool = []() -> HostSnapPool* {
        if (const char* v = std::getenv("FI_HOST_SNAP"); v && v[0] == '0') return nullptr;
        if (!cpu_ok()) return nullptr;
        return new HostSnapPool(default_workers());  // leaked with its detached workers
    }();
    return pool;
}

void HostSnapPool::submit(SnapJob* j) {
    if (j->height == 1) {
        j->lines_per_piece = 1;
        j->npieces = (j->width + kPieceElems - 1) / kPieceElems;
    } else {
        j->lines_per_piece = j->width >= kPieceElems ? 1 : kPieceElems / j->width;
        j->npieces = (j->height + j->lines_per_piece - 1) / j->lines_per_piece;
    }
    j->next.store(0);
    j->done.store(0);
    PoolState& st = state();
    {
        std::lock_guard<std::mutex> lk(st.mu);
        st.q.push_back(j);
    }
    st.cv.notify_all();
}

bool HostSnapPool::run_one() {
    PoolState& st = state();
    SnapJob* j = nullptr;
    long p = 0;
    {
        std::lock_guard<std::mutex> lk(st.mu);
        while (!st.q.empty()) {
            SnapJob* f = st.q.front();
            p = f->next.fetch_add(1);
            if (p < f->npieces) {
                j = f;
                break;
            }
            st.q.pop_front();  // every piece claimed
        }
    }
    if (!j) return false;
    convert_piece(j, p);
    _mm_sfence();  // streaming stores drained before the piece counts as done
    j->done.fetch_add(1, std::memory_order_release);
    return true;
}

void HostSnapPool::worker() {
    PoolState& st = state();
    for (;;) {
        if (run_one()) continue;
        std::unique_lock<std::mutex> lk(st.mu);
        st.cv.wait(lk, [&] { return !st.q.empty(); });
    }
}

void HostSnapPool::wait(SnapJob* j) {
    // help with this job's own pieces only: a piece of a later job would delay
    // the caller's next copy enqueue by a whole piece
    while (j->done.load(std::memory_order_acquire) < j->npieces) {
        const long p = j->next.fetch_add(1);
        if (p < j->npieces) {
            convert_piece(j, p);
            _mm_sfence();
            j->done.fetch_add(1, std::memory_order_release);
        } else {
            _mm_pause();
        }
    }
    // the caller may destroy the job now: drop it from the queue if no one has
    PoolState& st = state();
    std::lock_guard<std::mutex> lk(st.mu);
    for (auto it = st.q.begin(); it != st.q.end(); ++it)
        if (*it == j) {
            st.q.erase(it);
            break;
        }
}

}  // namespace fireiron::rt
