// tsg_bitpack.cu -- standalone bit-parallel kernels behind the bitpack API
// (bitpack.py:81-300).  They use the same encoder and the same recurrence as
// the engine path; the words are uint64 in the reference's numpy layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/tsg.h"
#include "tsg_kernels.cuh"

using namespace tsg;

extern "C" const char* tsg_last_error(void);

namespace {

int fail2(int code, const char* fmt, ...);

struct Buf {
    void* p = nullptr;
    ~Buf() { if (p) cudaFree(p); }
};

#define CK2(call)                                                                           \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) return fail2(TSG_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

__global__ void k_unpack_lanes(const LaneEntry<uint64_t>* lane, int64_t n, uint64_t* t, uint64_t* s) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) { t[i] = lane[i].t; s[i] = lane[i].s; }
}

// build_aggregate_batch from packed uint64 words [G][V+1] (bitpack.py:152-167, 211-244)
__global__ void k_aggregate(const uint64_t* __restrict__ T, const uint64_t* __restrict__ S,
                            const int32_t* __restrict__ lanes, int32_t G, int64_t nv,
                            uint64_t* cbt, uint64_t* cbf, uint64_t* cbu) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        uint64_t a = 0, b = 0, c = 0;
        if (v != 0) {
            for (int g = 0; g < G; ++g) {
                uint64_t bit = 1ull << g;
                if (lanes[g] == 0) { c |= bit; continue; }
                uint64_t t = T[(int64_t)g * nv + v], s = S[(int64_t)g * nv + v];
                uint64_t m = width_mask<uint64_t>(lanes[g]);
                if (t) a |= bit;
                if (s & ~t) b |= bit;
                if (~s & m) c |= bit;
            }
        }
        cbt[v] = a; cbf[v] = b; cbu[v] = c;
    }
}

// assignment_trigger (bitpack.py:120-135) over many clauses
__global__ void k_lane_trigger(const uint64_t* __restrict__ T, const uint64_t* __restrict__ S, uint64_t all,
                               uint64_t lane_mask, const int32_t* __restrict__ lits,
                               const int64_t* __restrict__ off, int64_t n, uint64_t* out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t af = all, ou = 0;
        for (int64_t j = off[i]; j < off[i + 1]; ++j) {
            int32_t lit = lits[j];
            int64_t v = lit < 0 ? -(int64_t)lit : lit;
            uint64_t t = T[v], s = S[v];
            step<uint64_t>(af, ou, lit > 0 ? (s & ~t) : (s & t), ~s);
        }
        out[i] = (af | ou) & lane_mask;
    }
}

// aggregate_trigger (bitpack.py:247-271) over many clauses
__global__ void k_agg_trigger(const uint64_t* __restrict__ cbt, const uint64_t* __restrict__ cbf,
                              const uint64_t* __restrict__ cbu, uint64_t all, uint64_t group_mask,
                              const int32_t* __restrict__ lits, const int64_t* __restrict__ off, int64_t n,
                              uint64_t* out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t af = all, ou = 0;
        for (int64_t j = off[i]; j < off[i + 1]; ++j) {
            int32_t lit = lits[j];
            int64_t v = lit < 0 ? -(int64_t)lit : lit;
            step<uint64_t>(af, ou, lit > 0 ? cbf[v] : cbt[v], cbu[v]);
        }
        out[i] = (af | ou) & group_mask;
    }
}

int set_device(int32_t device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail2(TSG_ECUDA, "no CUDA device");
    if (device < 0 || device >= n) return fail2(TSG_EINVAL, "device %d out of range", device);
    CK2(cudaSetDevice(device));
    return TSG_OK;
}

int check_lits(const int32_t* lits, const int64_t* off, int64_t n, int32_t num_vars) {
    for (int64_t j = 0; j < (n ? off[n] : 0); ++j) {
        int64_t v = lits[j] < 0 ? -(int64_t)lits[j] : lits[j];
        if (v > num_vars) return fail2(TSG_ERANGE, "literal %d out of range for %d variables", lits[j], num_vars);
    }
    return TSG_OK;
}

template <class T>
int upload(Buf& b, const T* src, int64_t n) {
    CK2(cudaMalloc(&b.p, std::max<int64_t>(n, 1) * sizeof(T)));
    if (n) CK2(cudaMemcpy(b.p, src, n * sizeof(T), cudaMemcpyHostToDevice));
    return TSG_OK;
}

int grid(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 8); }

}  // namespace

// error slot shared with tsg_engine.cu
extern "C" void tsg__set_error(const char* msg);

namespace {
int fail2(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    tsg__set_error(buf);
    return code;
}
}  // namespace

extern "C" {

int tsg_pack(int32_t device, const int8_t* rows, int64_t n, int64_t row_pitch, int32_t num_vars,
             int32_t lane_width, uint64_t* is_true, uint64_t* is_set) {
    if (lane_width < 1 || lane_width > 64) return fail2(TSG_EINVAL, "lane_width must be in 1..64, got %d", lane_width);
    if (n > lane_width) return fail2(TSG_ECAPACITY, "%lld assignments exceed lane width %d", (long long)n, lane_width);
    if (num_vars < 0) return fail2(TSG_EINVAL, "num_vars < 0");
    if (n > 0 && row_pitch < num_vars + 1) return fail2(TSG_EINVAL, "row pitch < num_vars+1");
    int r = set_device(device);
    if (r) return r;
    int64_t pitch = (num_vars + 1 + 15) / 16 * 16;
    Buf d_rows, d_lane;
    CK2(cudaMalloc(&d_rows.p, std::max<int64_t>(pitch * n, 16)));
    CK2(cudaMemset(d_rows.p, 0, std::max<int64_t>(pitch * n, 16)));
    if (n) CK2(cudaMemcpy2D(d_rows.p, pitch, rows, row_pitch, num_vars + 1, n, cudaMemcpyHostToDevice));
    int64_t nv2 = (int64_t)num_vars + 2;
    const int64_t vstride = (nv2 + 3) / 4 * 4;
    const int64_t lane_bytes = (vstride * (int64_t)sizeof(LaneEntry<uint64_t>) + 255) / 256 * 256;
    CK2(cudaMalloc(&d_lane.p, lane_bytes + nv2 * sizeof(AggEntry<uint64_t>)));
    EncodeChunk c{};
    c.G = 1;
    c.num_vars = num_vars;
    c.pitch = pitch;
    c.vstride = vstride;
    c.polarity = nullptr;
    c.row0[0] = 0;
    c.lanes[0] = (int32_t)n;
    auto* lane = (LaneEntry<uint64_t>*)d_lane.p;
    auto* agg = (AggEntry<uint64_t>*)((char*)d_lane.p + lane_bytes);
    k_encode<uint64_t, uint64_t><<<(unsigned)((nv2 + 127) / 128), dim3(32, 8)>>>((const int8_t*)d_rows.p, c, lane, agg);
    CK2(cudaGetLastError());
    Buf d_t, d_s;
    CK2(cudaMalloc(&d_t.p, (num_vars + 1) * 8));
    CK2(cudaMalloc(&d_s.p, (num_vars + 1) * 8));
    k_unpack_lanes<<<grid(num_vars + 1), 256>>>(lane, num_vars + 1, (uint64_t*)d_t.p, (uint64_t*)d_s.p);
    CK2(cudaGetLastError());
    CK2(cudaMemcpy(is_true, d_t.p, (num_vars + 1) * 8, cudaMemcpyDeviceToHost));
    CK2(cudaMemcpy(is_set, d_s.p, (num_vars + 1) * 8, cudaMemcpyDeviceToHost));
    return TSG_OK;
}

int tsg_aggregate(int32_t device, const uint64_t* is_true, const uint64_t* is_set, const int32_t* lane_counts,
                  int32_t n_groups, int32_t num_vars, int32_t group_width, uint64_t* cbt, uint64_t* cbf,
                  uint64_t* cbu) {
    if (group_width < 1 || group_width > 64) return fail2(TSG_EINVAL, "group_width must be in 1..64, got %d", group_width);
    if (n_groups > group_width) return fail2(TSG_ECAPACITY, "%d groups exceed group width %d", n_groups, group_width);
    int r = set_device(device);
    if (r) return r;
    int64_t nv = (int64_t)num_vars + 1;
    Buf T, S, L, O;
    if ((r = upload(T, is_true, nv * n_groups))) return r;
    if ((r = upload(S, is_set, nv * n_groups))) return r;
    if ((r = upload(L, lane_counts, n_groups))) return r;
    CK2(cudaMalloc(&O.p, nv * 3 * 8));
    uint64_t* o = (uint64_t*)O.p;
    k_aggregate<<<grid(nv), 256>>>((const uint64_t*)T.p, (const uint64_t*)S.p, (const int32_t*)L.p, n_groups, nv,
                                   o, o + nv, o + 2 * nv);
    CK2(cudaGetLastError());
    CK2(cudaMemcpy(cbt, o, nv * 8, cudaMemcpyDeviceToHost));
    CK2(cudaMemcpy(cbf, o + nv, nv * 8, cudaMemcpyDeviceToHost));
    CK2(cudaMemcpy(cbu, o + 2 * nv, nv * 8, cudaMemcpyDeviceToHost));
    return TSG_OK;
}

int tsg_lane_trigger(int32_t device, const uint64_t* is_true, const uint64_t* is_set, int32_t num_vars,
                     int32_t lane_width, uint64_t lane_mask, const int32_t* lits, const int64_t* offsets,
                     int64_t n, uint64_t* masks) {
    if (lane_width < 1 || lane_width > 64) return fail2(TSG_EINVAL, "lane_width must be in 1..64, got %d", lane_width);
    int r = check_lits(lits, offsets, n, num_vars);
    if (r) return r;
    if (n <= 0) return TSG_OK;
    if ((r = set_device(device))) return r;
    int64_t nv = (int64_t)num_vars + 1;
    Buf T, S, Lt, Of, O;
    if ((r = upload(T, is_true, nv))) return r;
    if ((r = upload(S, is_set, nv))) return r;
    if ((r = upload(Lt, lits, offsets[n]))) return r;
    if ((r = upload(Of, offsets, n + 1))) return r;
    CK2(cudaMalloc(&O.p, n * 8));
    k_lane_trigger<<<grid(n), 256>>>((const uint64_t*)T.p, (const uint64_t*)S.p, width_mask<uint64_t>(lane_width),
                                     lane_mask, (const int32_t*)Lt.p, (const int64_t*)Of.p, n, (uint64_t*)O.p);
    CK2(cudaGetLastError());
    CK2(cudaMemcpy(masks, O.p, n * 8, cudaMemcpyDeviceToHost));
    return TSG_OK;
}

int tsg_aggregate_trigger(int32_t device, const uint64_t* cbt, const uint64_t* cbf, const uint64_t* cbu,
                          int32_t num_vars, int32_t group_width, int32_t group_count, const int32_t* lits,
                          const int64_t* offsets, int64_t n, uint64_t* words) {
    if (group_width < 1 || group_width > 64) return fail2(TSG_EINVAL, "group_width must be in 1..64, got %d", group_width);
    int r = check_lits(lits, offsets, n, num_vars);
    if (r) return r;
    if (n <= 0) return TSG_OK;
    if (group_count == 0) {  // bitpack.py:259-260
        for (int64_t i = 0; i < n; ++i) words[i] = 0;
        return TSG_OK;
    }
    if ((r = set_device(device))) return r;
    int64_t nv = (int64_t)num_vars + 1;
    Buf A, B, Cc, Lt, Of, O;
    if ((r = upload(A, cbt, nv))) return r;
    if ((r = upload(B, cbf, nv))) return r;
    if ((r = upload(Cc, cbu, nv))) return r;
    if ((r = upload(Lt, lits, offsets[n]))) return r;
    if ((r = upload(Of, offsets, n + 1))) return r;
    CK2(cudaMalloc(&O.p, n * 8));
    k_agg_trigger<<<grid(n), 256>>>((const uint64_t*)A.p, (const uint64_t*)B.p, (const uint64_t*)Cc.p,
                                    width_mask<uint64_t>(group_width), width_mask<uint64_t>(group_count),
                                    (const int32_t*)Lt.p, (const int64_t*)Of.p, n, (uint64_t*)O.p);
    CK2(cudaGetLastError());
    CK2(cudaMemcpy(words, O.p, n * 8, cudaMemcpyDeviceToHost));
    return TSG_OK;
}

}  // extern "C"
