// Internal host-side declarations shared by the translation units of
// libshiftsolve_b200.so.  Not part of the public ABI (see include/).
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/shiftsolve_b200.h"

namespace ss {

// Greedy annihilation plan in device-friendly form: one packed word per
// rotation (r | c1 << 8 | c2 << 16, 1-based, as schedule.py stores them) and
// the exclusive prefix of job sizes (step t owns rotations
// [job_off[t], job_off[t+1])).
struct Sched {
    int nr = 0, nc = 0, steps = 0, rots = 0, max_job = 0;
    std::vector<uint32_t> rot;      // host copy
    std::vector<int32_t> job_off;   // host copy, steps+1 entries
    uint32_t* d_rot = nullptr;      // device copies
    int32_t* d_job_off = nullptr;
};

// Host greedy schedule (schedule.py:88-159), triplets 1-based.
int greedy_schedule(int n_rows, int n_cols, std::vector<int64_t>& job,
                    std::vector<int64_t>& info);

enum Phase { PH_REDUCTION = 0, PH_RQ = 1, PH_BATCHED_GEMM = 2, PH_OUTER_GEMM = 3, PH_TAIL = 4 };

// Pseudo-phase of k_update: it fuses the reference's batched GEMM and outer
// GEMM; its time is split between the two by their flop shares.
constexpr int PH_UPDATE = 100;

// One timed kernel (or kernel group) awaiting resolution.
struct TimeRec {
    int phase;
    cudaEvent_t a, b;
    double fl_batched, fl_outer;  // reference flops (for the update split)
    double fl_alg;                // algorithmic flops (roofline accounting)
};

}  // namespace ss

struct ss_handle {
    int device = 0;
    int num_sms = 148;
    size_t smem_optin = 0;
    std::string err;
    // grow-only device workspace
    void* ws = nullptr;
    size_t ws_bytes = 0;
    void* ws2 = nullptr;  // second workspace (reduction)
    size_t ws2_bytes = 0;
    double* d_scal = nullptr;  // [fro2, trace, scratch...]
    std::map<std::pair<int, int>, ss::Sched> sched;
    // accounting
    int timing = 0;
    double sec[5] = {0, 0, 0, 0, 0};
    double flops[5] = {0, 0, 0, 0, 0};
    int64_t launches = 0;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;  // fork / join events
    cudaStream_t aux_stream = nullptr;             // second stream of the sweep
    cudaStream_t copy_stream = nullptr;            // streamed H2D of Ahat (ss_tf_eval_stream)
    std::vector<cudaEvent_t> chunk_ev;             // one per streamed column chunk
    // deferred event timing (ss_set_timing): resolved by ss_phase_stats
    std::vector<cudaEvent_t> ev_pool;
    std::vector<ss::TimeRec> pending;
    int64_t upd_launches = 0;  // dominant kernel (k_update) live statistics
    double upd_sec = 0.0, upd_alg = 0.0;
};

namespace ss {

// cudaFuncSetAttribute acts on the current device: the launch helpers keep
// one "configured" bit per device (handles on several devices in one
// process; ss_create rejects device ids >= 64).  Atomic: handles are per
// thread, so first calls may race; configuring twice is harmless.
struct DevMask {
    std::atomic<uint64_t> bits{0};
    bool has(const ss_handle* h) const;
    void set(const ss_handle* h);
};
inline bool DevMask::has(const ss_handle* h) const {
    return (bits.load(std::memory_order_acquire) >> h->device) & 1u;
}
inline void DevMask::set(const ss_handle* h) {
    bits.fetch_or(uint64_t(1) << h->device, std::memory_order_acq_rel);
}

// Makes the handle's device current for one entry point and restores the
// caller's device on return.
struct DevGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DevGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        err = cudaSetDevice(device);
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int set_err(ss_handle* h, int code, const std::string& msg);
int cuda_err(ss_handle* h, cudaError_t e, const char* what);
// Ensure workspace of at least `bytes`; which=0 main, 1 secondary.
int ensure_ws(ss_handle* h, size_t bytes, int which = 0);
// Cached device schedule for (nr, nc).
const Sched* get_sched(ss_handle* h, int nr, int nc);
// Deferred event timing helpers (no-ops unless h->timing).
cudaEvent_t timing_begin(ss_handle* h, cudaStream_t st);
void timing_end(ss_handle* h, cudaStream_t st, cudaEvent_t a, int phase, double fl_batched = 0.0,
                double fl_outer = 0.0, double fl_alg = 0.0);
void timing_resolve(ss_handle* h);
// ||A||_F^2, trace(A) -> h->d_scal[0:2] (ss_sweep.cu)
int fro2_trace(ss_handle* h, int n, const double* A, int64_t lda, cudaStream_t st);

}  // namespace ss

#define SS_CUDA_TRY(h, expr)                                   \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return ss::cuda_err(h, _e, #expr); \
    } while (0)

#define SS_STR2(x) #x
#define SS_STR(x) SS_STR2(x)
#define SS_LAUNCH_CHECK(h)                                     \
    do {                                                       \
        (h)->launches++;                                       \
        cudaError_t _e = cudaGetLastError();                   \
        if (_e != cudaSuccess) return ss::cuda_err(h, _e, "kernel launch at " __FILE__ ":" SS_STR(__LINE__)); \
    } while (0)
