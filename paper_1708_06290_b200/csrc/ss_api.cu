// Handle lifecycle, errors, workspace, cached annihilation schedules and
// phase accounting for libshiftsolve_b200.so.
#include <cstdio>
#include <cstring>

#include "ss_internal.h"

namespace ss {

int set_err(ss_handle* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    return code;
}

int cuda_err(ss_handle* h, cudaError_t e, const char* what) {
    std::string msg = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return set_err(h, e == cudaErrorMemoryAllocation ? SS_ENOMEM : SS_ECUDA, msg);
}

int ensure_ws(ss_handle* h, size_t bytes, int which) {
    void** p = which ? &h->ws2 : &h->ws;
    size_t* cap = which ? &h->ws2_bytes : &h->ws_bytes;
    if (*cap >= bytes) return SS_OK;
    if (*p) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_err(h, e, "cudaDeviceSynchronize");
        cudaFree(*p);
        *p = nullptr;
        *cap = 0;
    }
    size_t want = bytes + (bytes >> 3);  // headroom: grow rarely
    cudaError_t e = cudaMalloc(p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            *p = nullptr;
            char buf[128];
            snprintf(buf, sizeof buf, "workspace allocation of %zu bytes failed", bytes);
            return set_err(h, SS_ENOMEM, buf);
        }
        want = bytes;
    }
    *cap = want;
    return SS_OK;
}

// schedule.py:88-159 greedy plan.  Positions (r, c), 1-based, c in
// [r, r+delta]; a target is zeroed against the rightmost ready+available
// helper of its row; zeroing (r, c) makes (r-1, c) available one step
// later; helpers rest for one step.  Rows are scanned bottom-up and targets
// left-to-right, exactly as the reference, so the plan is identical.
int greedy_schedule(int n_rows, int n_cols, std::vector<int64_t>& job,
                    std::vector<int64_t>& info) {
    job.clear();
    info.clear();
    if (n_rows < 1 || n_cols < n_rows) return -1;
    const int delta = n_cols - n_rows, w = delta + 1;
    auto at = [w](int r, int c) { return (r - 1) * w + (c - r); };
    std::vector<char> ready((size_t)n_rows * w, 1), avail((size_t)n_rows * w, 0);
    for (int r = 1; r <= n_rows; ++r)
        for (int c = r; c <= r + delta; ++c) avail[at(r, c)] = (r == n_rows) || (c == r);
    std::vector<int> resting, promoted;
    for (;;) {
        for (int p : resting) ready[p] = 1;
        resting.clear();
        for (int p : promoted) avail[p] = 1;
        promoted.clear();
        int count = 0;
        for (int r = n_rows; r >= 1; --r) {
            for (int c1 = r; c1 <= r + delta; ++c1) {
                const int p1 = at(r, c1);
                if (!(ready[p1] && avail[p1])) continue;
                for (int c2 = r + delta; c2 > c1; --c2) {
                    const int p2 = at(r, c2);
                    if (!(ready[p2] && avail[p2])) continue;
                    info.push_back(r);
                    info.push_back(c1);
                    info.push_back(c2);
                    ++count;
                    ready[p1] = ready[p2] = 0;
                    resting.push_back(p2);
                    if (r > 1) {
                        const int pu = at(r - 1, c1);
                        avail[pu] = 0;
                        promoted.push_back(pu);
                    }
                    break;
                }
            }
        }
        if (count == 0) break;
        job.push_back(count);
    }
    return (int)job.size();
}

const Sched* get_sched(ss_handle* h, int nr, int nc) {
    auto key = std::make_pair(nr, nc);
    auto it = h->sched.find(key);
    if (it != h->sched.end()) return &it->second;
    std::vector<int64_t> job, info;
    if (greedy_schedule(nr, nc, job, info) < 0) return nullptr;
    Sched s;
    s.nr = nr;
    s.nc = nc;
    s.steps = (int)job.size();
    s.rots = (int)(info.size() / 3);
    s.job_off.resize(s.steps + 1);
    s.job_off[0] = 0;
    for (int t = 0; t < s.steps; ++t) {
        s.job_off[t + 1] = s.job_off[t] + (int32_t)job[t];
        if (job[t] > s.max_job) s.max_job = (int)job[t];
    }
    s.rot.resize(s.rots);
    for (int q = 0; q < s.rots; ++q)
        s.rot[q] = (uint32_t)info[3 * q] | ((uint32_t)info[3 * q + 1] << 8) |
                   ((uint32_t)info[3 * q + 2] << 16);
    size_t nrot = s.rot.empty() ? 1 : s.rot.size();
    if (cudaMalloc(&s.d_rot, nrot * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&s.d_job_off, s.job_off.size() * sizeof(int32_t)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (!s.rot.empty())
        cudaMemcpy(s.d_rot, s.rot.data(), s.rot.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    cudaMemcpy(s.d_job_off, s.job_off.data(), s.job_off.size() * sizeof(int32_t),
               cudaMemcpyHostToDevice);
    auto res = h->sched.emplace(key, std::move(s));
    return &res.first->second;
}

static cudaEvent_t ev_get(ss_handle* h) {
    if (!h->ev_pool.empty()) {
        cudaEvent_t e = h->ev_pool.back();
        h->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

cudaEvent_t timing_begin(ss_handle* h, cudaStream_t st) {
    if (!h->timing) return nullptr;
    cudaEvent_t e = ev_get(h);
    cudaEventRecord(e, st);
    return e;
}

void timing_end(ss_handle* h, cudaStream_t st, cudaEvent_t a, int phase, double fl_batched,
                double fl_outer, double fl_alg) {
    if (!h->timing || !a) return;
    cudaEvent_t b = ev_get(h);
    cudaEventRecord(b, st);
    h->pending.push_back(TimeRec{phase, a, b, fl_batched, fl_outer, fl_alg});
}

void timing_resolve(ss_handle* h) {
    for (auto& r : h->pending) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        const double sec = ms * 1e-3;
        if (r.phase == PH_UPDATE) {
            const double tot = r.fl_batched + r.fl_outer;
            const double fr = tot > 0 ? r.fl_batched / tot : 0.0;
            h->sec[PH_BATCHED_GEMM] += sec * fr;
            h->sec[PH_OUTER_GEMM] += sec * (1.0 - fr);
            h->upd_launches++;
            h->upd_sec += sec;
            h->upd_alg += r.fl_alg;
        } else if (r.phase >= 0 && r.phase < 5) {
            h->sec[r.phase] += sec;
        }
        h->ev_pool.push_back(r.a);
        h->ev_pool.push_back(r.b);
    }
    h->pending.clear();
}

}  // namespace ss

extern "C" {

int ss_version(void) { return 100; }  // 0.1.0

int ss_create(ss_handle** out, int device) {
    if (!out) return SS_EARG;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev || device >= 64) {
        cudaGetLastError();
        return SS_ECUDA;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return SS_ECUDA;
    ss_handle* h = new ss_handle();
    h->device = device;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    h->smem_optin = (size_t)optin;
    if (cudaMalloc(&h->d_scal, 64 * sizeof(double)) != cudaSuccess ||
        cudaEventCreate(&h->ev_a) != cudaSuccess || cudaEventCreate(&h->ev_b) != cudaSuccess) {
        cudaGetLastError();
        delete h;
        cudaSetDevice(prev);
        return SS_ECUDA;
    }
    cudaSetDevice(prev);  // the caller's current device is left as it was
    *out = h;
    return SS_OK;
}

void ss_destroy(ss_handle* h) {
    if (!h) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (auto& kv : h->sched) {
        cudaFree(kv.second.d_rot);
        cudaFree(kv.second.d_job_off);
    }
    if (h->ws) cudaFree(h->ws);
    if (h->ws2) cudaFree(h->ws2);
    if (h->d_scal) cudaFree(h->d_scal);
    for (auto& r : h->pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    if (h->aux_stream) cudaStreamDestroy(h->aux_stream);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    for (auto e : h->chunk_ev) cudaEventDestroy(e);
    if (h->ev_a) cudaEventDestroy(h->ev_a);
    if (h->ev_b) cudaEventDestroy(h->ev_b);
    delete h;
    cudaSetDevice(prev);
}

const char* ss_last_error(const ss_handle* h) { return h ? h->err.c_str() : "null handle"; }

int ss_greedy_schedule(int n_rows, int n_cols, int64_t* job_size, int64_t job_cap,
                       int64_t* rot_info, int64_t info_cap, int* num_steps, int* num_rots) {
    std::vector<int64_t> job, info;
    int steps = ss::greedy_schedule(n_rows, n_cols, job, info);
    if (steps < 0) return SS_EDIM;
    if ((int64_t)job.size() > job_cap || (int64_t)info.size() > info_cap) return SS_EARG;
    if (!job.empty()) memcpy(job_size, job.data(), job.size() * sizeof(int64_t));
    if (!info.empty()) memcpy(rot_info, info.data(), info.size() * sizeof(int64_t));
    if (num_steps) *num_steps = steps;
    if (num_rots) *num_rots = (int)(info.size() / 3);
    return SS_OK;
}

int ss_set_timing(ss_handle* h, int enabled) {
    if (!h) return SS_EARG;
    h->timing = enabled ? 1 : 0;
    return SS_OK;
}

int ss_phase_stats(ss_handle* h, double* seconds5, double* flops5) {
    if (!h) return SS_EARG;
    ss::timing_resolve(h);
    for (int i = 0; i < 5; ++i) {
        if (seconds5) seconds5[i] = h->sec[i];
        if (flops5) flops5[i] = h->flops[i];
    }
    return SS_OK;
}

void ss_reset_stats(ss_handle* h) {
    if (!h) return;
    ss::timing_resolve(h);
    for (int i = 0; i < 5; ++i) h->sec[i] = h->flops[i] = 0.0;
    h->upd_launches = 0;
    h->upd_sec = h->upd_alg = 0.0;
}

int ss_update_kernel_stats(ss_handle* h, int64_t* launches, double* seconds, double* alg_flops) {
    if (!h) return SS_EARG;
    ss::timing_resolve(h);
    if (launches) *launches = h->upd_launches;
    if (seconds) *seconds = h->upd_sec;
    if (alg_flops) *alg_flops = h->upd_alg;
    return SS_OK;
}

int64_t ss_launch_count(const ss_handle* h) { return h ? h->launches : 0; }

}  // extern "C"
