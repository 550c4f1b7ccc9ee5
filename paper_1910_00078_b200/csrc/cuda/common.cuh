// Shared device helpers for the primkit-b200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "kernels.h"

namespace pk {

// Process-wide count of kernels launched by this library (pk_cuda_launch_count).
void count_launch(int n = 1);
// Appends the kernel's template instance to the thread's variant log (pk_cuda_variant).
void note_kernel(const void* fn);
// Kernel choice in force for the calling thread's current top-level launcher
// (set by pk_cuda_igemm_tc_fwd / _dgrad / _wgrad from their config argument,
// read by the family dispatchers below them); nullptr = heuristics only.
const pk_tc_config* active_tc_config();
struct ActiveTcConfig {
    explicit ActiveTcConfig(const pk_tc_config* c);
    ~ActiveTcConfig();
    const pk_tc_config* prev;
};
inline int cfg_field(int pk_tc_config::*f) {
    const pk_tc_config* c = active_tc_config();
    return c ? c->*f : 0;
}

template <typename T>
struct Elt;
template <>
struct Elt<float> {
    static __device__ __forceinline__ float load(const float* p) { return *p; }
    static __device__ __forceinline__ void store(float* p, float v) { *p = v; }
};
template <>
struct Elt<__nv_bfloat16> {
    static __device__ __forceinline__ float load(const __nv_bfloat16* p) {
        return __bfloat162float(*p);
    }
    // Round-to-nearest-even, the reference's round_bf16 (tensor.cpp:44-54)
    // for every non-NaN input.
    static __device__ __forceinline__ void store(__nv_bfloat16* p, float v) {
        *p = __float2bfloat16_rn(v);
    }
};

template <typename T>
__device__ __forceinline__ float ld(const T* p) { return Elt<T>::load(p); }
template <typename T>
__device__ __forceinline__ void st(T* p, float v) { Elt<T>::store(p, v); }

// The reference's activation_apply (primitives.cpp:154-164).
__device__ __forceinline__ float activate(int act, float alpha, float v) {
    switch (act) {
        case 0: return v > 0.0f ? v : 0.0f;
        case 1: return v > 0.0f ? v : alpha * v;
        case 2: return 1.0f / (1.0f + expf(-v));
        case 3: return tanhf(v);
        default: return v;
    }
}

// Fusion epilogue on one fp32 accumulator for output channel k at output
// pixel (oh, ow) of a P x Q image (fusion.cpp:384-398 order).
__device__ __forceinline__ float apply_epilogue(const pk_epilogue& e, float acc, int k, int oh,
                                                int ow, int P, int Q) {
    if (e.bias) acc += e.bias[k];
    if (e.bn_mean) {
        const int bi = e.bn_per_activation ? (k * P + oh) * Q + ow : k;
        if (e.bn_standalone) {
            const float inv = 1.0f / sqrtf(e.bn_var[bi] + e.bn_eps);
            acc = e.bn_gamma[bi] * (acc - e.bn_mean[bi]) * inv + e.bn_beta[bi];
        } else {
            acc = (acc - e.bn_mean[bi]) / sqrtf(e.bn_var[bi] + e.bn_eps) * e.bn_gamma[bi] +
                  e.bn_beta[bi];
        }
    }
    if (e.act >= 0) acc = activate(e.act, e.act_alpha, acc);
    return acc;
}

__host__ __device__ inline bool epilogue_active(const pk_epilogue* e) {
    return e && (e->bias || e->bn_mean || e->act >= 0 || e->ch_scale);
}

// Activation on the tensor-core epilogue path (bf16 outputs): ReLU/LeakyReLU
// exactly as the reference; sigmoid/tanh through the MUFU exp2 unit (relative
// error ~1e-6, far below the bf16 output rounding) so the unrolled epilogue
// stays compact in the instruction cache.
__device__ __forceinline__ float activate_fast(int act, float alpha, float v) {
    switch (act) {
        case 0: return v > 0.0f ? v : 0.0f;
        case 1: return v > 0.0f ? v : alpha * v;
        case 2: return __frcp_rn(1.0f + __expf(-v));
        case 3: return 2.0f * __frcp_rn(1.0f + __expf(-2.0f * v)) - 1.0f;
        default: return v;
    }
}

// Fused epilogue for 64 consecutive output channels [ch0, ch0 + 64) of one
// output pixel (oy, ox) of a P x Q image, in place on fp32 accumulators.
// ch_scale / ch_shift must be readable up to ch0 + 64 (host pads them);
// the unfolded form only touches channels below n_out.
__device__ __forceinline__ void epilogue_chunk64(const pk_epilogue& e, float (&x)[64], int ch0,
                                                 int n_out, int oy, int ox, int P, int Q) {
    if (e.ch_scale) {
        const float4* sc = reinterpret_cast<const float4*>(e.ch_scale + ch0);
        const float4* sh = reinterpret_cast<const float4*>(e.ch_shift + ch0);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float4 s = __ldg(sc + j), t = __ldg(sh + j);
            x[4 * j + 0] = fmaf(x[4 * j + 0], s.x, t.x);
            x[4 * j + 1] = fmaf(x[4 * j + 1], s.y, t.y);
            x[4 * j + 2] = fmaf(x[4 * j + 2], s.z, t.z);
            x[4 * j + 3] = fmaf(x[4 * j + 3], s.w, t.w);
        }
    } else if (e.bias || e.bn_mean) {
        // general form (per-activation BN): rare, kept out of the fast path
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            float a = x[j];
            const int k = ch0 + j;
            if (k >= n_out) continue;
            if (e.bias) a += __ldg(e.bias + k);
            if (e.bn_mean) {
                const int bi = e.bn_per_activation ? (k * P + oy) * Q + ox : k;
                a = (a - __ldg(e.bn_mean + bi)) / sqrtf(__ldg(e.bn_var + bi) + e.bn_eps) *
                        __ldg(e.bn_gamma + bi) +
                    __ldg(e.bn_beta + bi);
            }
            x[j] = a;
        }
    }
    const float alpha = e.act_alpha;
    if (e.act == 0) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(0, alpha, x[j]);
    } else if (e.act == 1) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(1, alpha, x[j]);
    } else if (e.act == 2) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(2, alpha, x[j]);
    } else if (e.act == 3) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(3, alpha, x[j]);
    }
}

// Round a lane's 64 fp32 outputs to bf16 and stage them as one 128-byte row
// (16-byte chunks XOR-swizzled by lane & 7) for a TMA / coalesced store.
// Channels at or beyond `valid` are written as zero; the common full chunk
// takes the mask-free path (the per-element selects cost 3x the packing).
__device__ __forceinline__ uint32_t pack2(float a, float b, bool f16) {
    if (f16) {
        __half2 h2 = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h2);
    }
    __nv_bfloat162 b2 = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&b2);
}

// f16: stage IEEE fp16 instead of bf16 (the fp16 transform domain of the
// tensor-core Winograd, winograd_tc.cu).
__device__ __forceinline__ void pack_stage64(const float (&xf)[64], uint32_t stg_u, int lane,
                                             int valid, bool f16 = false) {
    if (f16) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = jj * 8 + 2 * e;
                w[e] = pack2(c < valid ? xf[c] : 0.0f, c + 1 < valid ? xf[c + 1] : 0.0f, true);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg_u + lane * 128 + ((jj ^ (lane & 7)) << 4)),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
        }
        return;
    }
    if (valid >= 64) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 b2 = __floats2bfloat162_rn(xf[jj * 8 + 2 * e], xf[jj * 8 + 2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t*>(&b2);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg_u + lane * 128 + ((jj ^ (lane & 7)) << 4)),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
        }
    } else {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = jj * 8 + 2 * e;
                __nv_bfloat162 b2 = __floats2bfloat162_rn(c < valid ? xf[c] : 0.0f,
                                                          c + 1 < valid ? xf[c + 1] : 0.0f);
                w[e] = *reinterpret_cast<uint32_t*>(&b2);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg_u + lane * 128 + ((jj ^ (lane & 7)) << 4)),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
        }
    }
}

// ---- batch-norm statistics in the tensor-core epilogues -------------------
// A staged tile is 32 rows x 64 channels of bf16 (128-byte rows, 16-byte
// chunks XOR-swizzled by row & 7). Lane l owns channels ch0 + 2l, ch0 + 2l + 1
// and sums them over the valid rows. Sums are kept in registers per channel
// block (persistent CTAs keep their channel block: 148 % n_tiles_n == 0 for
// n_tiles_n in {1, 2, 4}) and flushed to the CTA's slice of pk_epilogue.stats
// only when the block changes and at the end — one atomic per channel per
// CTA instead of one per tile.

__device__ __forceinline__ uint32_t staged_word(uint32_t stg_u, int r, int lane) {
    uint32_t wv;
    asm volatile("ld.shared.b32 %0, [%1];"
                 : "=r"(wv)
                 : "r"(stg_u + r * 128 + ((((lane >> 2) ^ (r & 7)) << 4) | ((lane & 3) << 2))));
    return wv;
}

// forward: (sum, sumsq) of the stored values for both channels of the lane.
// Packed f32x2 arithmetic (FADD2 / FFMA2): a bf16 pair widens to an f32 pair
// with two bit ops, then one add and one fma cover both channels.
__device__ __forceinline__ float4 stats64_fwd(uint32_t stg_u, int lane, unsigned ok) {
    unsigned long long sum = 0ull, sq = 0ull;  // (ch0, ch1) f32 pairs
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
        const uint32_t wv = staged_word(stg_u, r, lane);
        // rows past the tile (ok bit clear) contribute zeros
        const uint32_t w = ((ok >> r) & 1u) ? wv : 0u;
        unsigned long long f;
        asm("{\n\t.reg .b32 lo, hi;\n\tshl.b32 lo, %1, 16;\n\tand.b32 hi, %1, 0xffff0000;\n\t"
            "mov.b64 %0, {lo, hi};\n\t}"
            : "=l"(f)
            : "r"(w));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(sum) : "l"(f));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(sq) : "l"(f));
    }
    float4 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.z) : "l"(sum));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.y), "=f"(a.w) : "l"(sq));
    return a;
}

// backward (see pk_epilogue.bnb_*): (sum d, sum d*xhat) for both channels;
// y rows are fetched 8 at a time so the loads overlap
__device__ __forceinline__ float4 stats64_bwd(const pk_epilogue& e, uint32_t stg_u, int lane,
                                              unsigned ok, long long pix, int ch0, int n_out,
                                              int pitch) {
    const int ch = ch0 + 2 * lane;
    const bool v0 = ch < n_out, v1 = ch + 1 < n_out;
    const float g0 = v0 ? e.bnb_gamma[ch] : 0.f, g1 = v1 ? e.bnb_gamma[ch + 1] : 0.f;
    const float b0 = v0 ? e.bnb_beta[ch] : 0.f, b1 = v1 ? e.bnb_beta[ch + 1] : 0.f;
    const float m0 = v0 ? e.bnb_mean[ch] : 0.f, m1 = v1 ? e.bnb_mean[ch + 1] : 0.f;
    const float i0 = v0 ? e.bnb_invstd[ch] : 0.f, i1 = v1 ? e.bnb_invstd[ch + 1] : 0.f;
    const float sc0 = g0 * i0, sh0 = b0 - m0 * sc0, sc1 = g1 * i1, sh1 = b1 - m1 * sc1;
    const __nv_bfloat16* y = static_cast<const __nv_bfloat16*>(e.bnb_y);
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
    for (int r0 = 0; r0 < 32; r0 += 8) {
        uint32_t yv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long rp = __shfl_sync(0xffffffffu, pix, r0 + u);
            yv[u] = (v0 && ((ok >> (r0 + u)) & 1u))
                        ? __ldg(reinterpret_cast<const unsigned int*>(y + rp * pitch + ch))
                        : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int r = r0 + u;
            if (!((ok >> r) & 1u)) continue;
            const uint32_t wv = staged_word(stg_u, r, lane);
            const float2 dz = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv));
            const float2 yy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&yv[u]));
            float d0 = dz.x, d1 = dz.y;
            if (e.bnb_relu) {
                // the forward ReLU mask, recomputed exactly as bn_apply_bf16x8_kernel
                // does (folded affine, bn_fold in bn.cu)
                if (!(fmaf(yy.x, sc0, sh0) > 0.0f)) d0 = 0.f;
                if (!(fmaf(yy.y, sc1, sh1) > 0.0f)) d1 = 0.f;
            }
            a.x += d0;
            a.y = fmaf(d0, (yy.x - m0) * i0, a.y);
            a.z += d1;
            a.w = fmaf(d1, (yy.y - m1) * i1, a.w);
        }
    }
    return a;
}

struct BnStatAcc {
    int base[2];
    float4 a[2];
    __device__ __forceinline__ void init() {
        base[0] = base[1] = -1;
        a[0] = a[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __device__ __forceinline__ void flush(const pk_epilogue& e, int s, int lane, int n_out) {
        if (base[s] < 0) return;
        float* part = e.stats + (size_t)blockIdx.x * n_out * 2;
        const int ch = base[s] + 2 * lane;
        if (ch < n_out) {
            atomicAdd(part + 2 * ch, a[s].x);
            atomicAdd(part + 2 * ch + 1, a[s].y);
        }
        if (ch + 1 < n_out) {
            atomicAdd(part + 2 * ch + 2, a[s].z);
            atomicAdd(part + 2 * ch + 3, a[s].w);
        }
        a[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        base[s] = -1;
    }
    // slot: which of the warp's (at most two) channel blocks this chunk is
    __device__ __forceinline__ void add(const pk_epilogue& e, uint32_t stg_u, int lane, bool row_ok,
                                        long long pix, int slot, int ch0, int n_out, int pitch) {
        const unsigned ok = __ballot_sync(0xffffffffu, row_ok);
        if (base[slot] != ch0) {
            flush(e, slot, lane, n_out);
            base[slot] = ch0;
        }
        const float4 v = e.bnb_y ? stats64_bwd(e, stg_u, lane, ok, pix, ch0, n_out, pitch)
                                 : stats64_fwd(stg_u, lane, ok);
        a[slot].x += v.x;
        a[slot].y += v.y;
        a[slot].z += v.z;
        a[slot].w += v.w;
    }
    __device__ __forceinline__ void finish(const pk_epilogue& e, int lane, int n_out) {
        flush(e, 0, lane, n_out);
        flush(e, 1, lane, n_out);
    }
};

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// Programmatic dependent launch (PDL). Step kernels are launched with
// programmatic stream serialization, so kernel i+1 may be scheduled while
// kernel i drains: it runs its prologue (barrier init, TMEM alloc, tensor-map
// prefetch) and then blocks in pdl_wait() until kernel i has COMPLETED and its
// memory is visible. Every kernel launched through pk_launch calls pdl_wait()
// before its first global memory access, then pdl_trigger() so its own
// successor can be scheduled. Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();  // PK_PDL=0 disables (A/B comparisons)

// ---- in-kernel split-K finish (wgrad) ----------------------------------------
// The CTAs of a split-K wgrad grid each write an fp32 partial [split][total];
// instead of a separate sum launch, every CTA arrives on a grid barrier and then
// sums a slice of the output over all splits in FIXED split order (deterministic,
// bit-identical to wgrad_sum_kernel) and stores bf16. Only for grids whose CTAs
// are all co-resident (grid <= SMs, one CTA per SM): the host checks. sync[0]
// counts arrivals, sync[1] departures; the last CTA to leave resets both, so a
// slot is reusable by the next launch (stream-ordered) and by graph replays.
__device__ __forceinline__ void splitk_finish(const float* __restrict__ partial, int splits,
                                              long long total, __nv_bfloat16* __restrict__ dw,
                                              unsigned int* sync) {
    const unsigned nctas = gridDim.x * gridDim.y * gridDim.z;
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    __threadfence();  // this CTA's partial stores before its arrival
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(&sync[0], 1u);
        unsigned seen;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(sync) : "memory");
            if (seen < nctas) __nanosleep(64);
        } while (seen < nctas);
    }
    __syncthreads();
    const long long quads = total / 4;
    const long long per = (quads + nctas - 1) / nctas;
    const long long q0 = (long long)cta * per, q1 = q0 + per < quads ? q0 + per : quads;
    const float4* p = reinterpret_cast<const float4*>(partial);
    for (long long i = q0 + threadIdx.x; i < q1; i += blockDim.x) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int s = 0;
        for (; s + 8 <= splits; s += 8) {  // eight loads in flight, then the adds in order
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (size_t)(s + u) * quads + i);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                acc.x += v[u].x;
                acc.y += v[u].y;
                acc.z += v[u].z;
                acc.w += v[u].w;
            }
        }
        for (; s < splits; ++s) {
            const float4 v = __ldcg(p + (size_t)s * quads + i);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        const __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
        reinterpret_cast<uint2*>(dw)[i] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
    if (cta == 0)  // tail (total not a multiple of 4)
        for (long long i = quads * 4 + threadIdx.x; i < total; i += blockDim.x) {
            float a = 0.f;
            for (int s = 0; s < splits; ++s) a += __ldcg(partial + (size_t)s * total + i);
            dw[i] = __float2bfloat16_rn(a);
        }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&sync[1], 1u) == nctas - 1) {
        sync[0] = 0u;
        sync[1] = 0u;
        __threadfence();
    }
}
// A free barrier slot (round-robin over a static pool) or nullptr if unavailable.
unsigned int* splitk_sync_slot();

template <typename... KArgs, typename... Args>
cudaError_t pk_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    note_kernel(reinterpret_cast<const void*>(kern));
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// Same with a runtime cluster size along x (CTA pairs for cta_group::2 kernels).
template <typename... KArgs, typename... Args>
cudaError_t pk_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (cluster_x > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster_x;
        attr[na].val.clusterDim.y = 1;
        attr[na++].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    note_kernel(reinterpret_cast<const void*>(kern));
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace pk

// Dispatch on the storage element type.
#define PK_DISPATCH_DTYPE(dtype, T, ...)        \
    do {                                        \
        if ((dtype) == PK_BF16) {               \
            using T = __nv_bfloat16;            \
            __VA_ARGS__;                        \
        } else {                                \
            using T = float;                    \
            __VA_ARGS__;                        \
        }                                       \
    } while (0)
