// vrb_internal.cuh -- shared internals of libvrb.so (product path only; no
// code here is shared with oracle/).
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "../../include/vrb.h"

namespace vrb {

// ---------------------------------------------------------------------------
// Errors: internal code throws vrb::Error; the C ABI (vrb_api.cu) catches it,
// stores the message in the thread-local last-error slot and returns the code.
// ---------------------------------------------------------------------------
struct Error {
    vrb_status status;
    std::string msg;
};

[[noreturn]] void fail(vrb_status st, const char* fmt, ...);

#define VRB_CUDA(x)                                                                       \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess)                                                            \
            ::vrb::fail(VRB_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,                \
                        cudaGetErrorString(e_));                                          \
    } while (0)
// Every kernel launch is followed by VRB_LAUNCH_CHECK(), which also counts it
// (vrb_launch_count(): the bench's gpu_launches claim).
void count_launch();
#define VRB_LAUNCH_CHECK()              \
    do {                                \
        ::vrb::count_launch();          \
        VRB_CUDA(cudaGetLastError());   \
    } while (0)

// ---------------------------------------------------------------------------
// Device memory through the allocator hook (default cudaMallocAsync).
// ---------------------------------------------------------------------------
void* dalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, size_t bytes, cudaStream_t s);

template <class T>
class DBuf {
  public:
    DBuf() = default;
    DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
    ~DBuf() { reset(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { *this = std::move(o); }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p_ = o.p_; n_ = o.n_; s_ = o.s_;
            o.p_ = nullptr; o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t n, cudaStream_t s) {
        reset();
        n_ = n; s_ = s;
        p_ = n ? static_cast<T*>(dalloc(n * sizeof(T), s)) : nullptr;
    }
    void reset() {
        if (p_) dfree(p_, n_ * sizeof(T), s_);
        p_ = nullptr; n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }
    operator T*() const { return p_; }

  private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = 0;
};

// Owned output allocation recorded in a result handle, with the free hook in
// force when it was made (the hook may be changed before the handle is freed).
struct Alloc {
    void* p;
    size_t bytes;
    vrb_free_fn fn = nullptr;   // nullptr: cudaFreeAsync
    void* ctx = nullptr;
};
Alloc dalloc_owned(size_t bytes, cudaStream_t s);
void dfree_owned(const Alloc& a);

// ---------------------------------------------------------------------------
// Constants
// ---------------------------------------------------------------------------
constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr int kNumSMs = 148;            // B200; queried at run time where it matters
constexpr int64_t kMaxN = (int64_t)1 << 21;   // 21-bit vertex ids in packed lex codes

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int device_sm_count();
size_t device_max_smem_optin();

// ---------------------------------------------------------------------------
// Primitive launchers (scan.cu, radix_sort.cu)
// ---------------------------------------------------------------------------
// out[i] = sum_{q<i} in[q] for i in [0, n]; out has n + 1 entries.
void exclusive_scan(const uint32_t* in, uint64_t* out, int64_t n, cudaStream_t s);
void exclusive_scan(const uint64_t* in, uint64_t* out, int64_t n, cudaStream_t s);
// out[i] = sum_{q<=i} in[q] (u32 result; the caller guarantees no overflow)
void inclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s);
// out[i] = 1-based dense rank of sorted_keys[i] (the inclusive scan of the
// run-start flags, computed on the fly from the keys)
void dense_ranks(const uint64_t* sorted_keys, uint32_t* out, int64_t n, cudaStream_t s);

// Bitwise OR over i of (keys[i] ^ keys[0]): the key bits that vary.
uint64_t varying_bits(const uint64_t* keys, int64_t n, cudaStream_t s);

// (max - min) of the keys as a bit mask of its length (every key - min fits
// in it); *kmin = min.  A sort of (key - kmin) needs only those digits.
uint64_t key_range(const uint64_t* keys, int64_t n, cudaStream_t s, uint64_t* kmin,
                   const unsigned long long* reduced = nullptr);

// Stable ascending LSD radix sort of (keys, vals) on the bit range [0, 64)
// restricted to the 8-bit digits that contain a bit of `varying`.  Uses
// (keys_alt, vals_alt) as ping-pong space; returns true if the sorted result
// ended in the *_alt buffers.  With bias != 0 the sort key is (key - bias):
// the first pass subtracts it while loading, so the sorted keys are biased
// (*biased = true) unless no pass ran.
bool radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                      int64_t n, uint64_t varying, cudaStream_t s, uint64_t bias = 0, bool* biased = nullptr);

// The same sort on keys alone (8 bytes per item per pass instead of 12).
bool radix_sort_keys(uint64_t* keys, uint64_t* keys_alt, int64_t n, uint64_t varying, cudaStream_t s);

// Fill helpers
void fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t s);
void iota_u32(uint32_t* p, int64_t n, cudaStream_t s);

// Stage timing (vrb_set_profiling / vrb_last_stage_ms)
struct StageTimer {
    bool on = false;
    cudaStream_t s = 0;
    std::vector<std::pair<int, cudaEvent_t>> marks;
    bool nvtx_open = false;
    void start(cudaStream_t st);
    void begin(int stage);  // start of `stage` (NVTX range)
    void mark(int stage);   // end of `stage`
    void finish();          // synchronises and stores into the thread-local slot
    ~StageTimer();
};
bool profiling_enabled();

}  // namespace vrb
