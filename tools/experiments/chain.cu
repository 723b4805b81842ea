// chain.cu — the post-attention half of a layer as ONE persistent kernel at prompt sizes of one 128-row tile
// (the per-layer prefill compute; C2 = OPT-1.3B, T = 128):
//     job 0  O projection        h += attn · Wo^T + b        (split-K S0, residual epilogue)
//     job 1  norm 2              x = LN(h) | RMS(h)          (one row per item)
//     job 2  FC1 | gate·up       mlp = ReLU(x · W1^T + b) | SiLU(g)·u
//     job 3  FC2 | down          h += mlp · W2^T + b
// At M = 128 rows every projection is a weight stream (intensity 128 flop/B) that takes a few microseconds, so
// with one kernel per step the GPU spends a large share of the layer in launch, ramp-up and drain. Here the
// steps are work items of one launch that keep every SM streaming weights:
//   * items (job-major; a GEMM job's items are (output tile, K split) pairs, split-minor) are claimed from a
//     global counter by whichever CTA is free, so an item is only ever held by a running CTA and waits only for
//     items claimed before it: no co-residency assumption, no deadlock;
//   * a GEMM item's WEIGHT tiles are requested as soon as it is claimed — before the previous job has finished —
//     and only its activation tiles wait (acquire on the previous job's completion count), so the weight
//     stream of job j+1 overlaps the tail of job j;
//   * warp specialisation as in gemm_big_kernel: warp 0 TMA producer (claims items), warp 1 single-thread
//     tcgen05.mma issuer, warps 2-5 epilogue / norm; the claimed items flow to warps 1-5 through a 4-deep
//     shared-memory queue; two 128-column TMEM accumulators let item i's epilogue overlap item i+1's mainloop;
//   * split-K partials go to an L2-resident fp32 workspace ([col/4][row][4], coalesced); the LAST split to
//     arrive (acq_rel counter per tile) sums the S partials in the fixed order 0..S-1 and applies the epilogue,
//     so each output element is computed exactly as gemm_kernel<EPI, S> computes it (same K ranges, same MMA
//     order, same summation order, same epilogue expressions) and a norm row exactly as norm_kernel does
//     (rownorm.cuh): results are bit-identical to the per-op path;
//   * cross-CTA hand-off: writers fence the async proxy (the next job reads by TMA), a named barrier, then one
//     release increment; readers acquire, fence the async proxy, then issue TMA.
// The control words of a launch are left zeroed by its last CTA; consecutive launches rotate over
// kChainCtlSets sets so a launch that starts early (programmatic dependent launch) never sees the previous
// one's counters.
//
// MEASURED (B200, C2, tools/chain_trace.py, profiles/r01_chain_trace_C2.json): correct and bit-identical, but
// ~146 us per layer against ~60 us for the four per-op kernels it replaces, so it is opt-in (PB_CHAIN=1).
// Under load a dependent global-memory round trip costs 2-4 us here, and the split-K hand-off through L2
// (partial store -> arrival count -> the last split loads the other partials chunk by chunk -> residual
// read-modify-write -> publish) is a chain of ~8 of them per job: the finishing epilogue alone takes 18-25 us,
// where the per-op kernel reduces through distributed shared memory inside its cluster in ~1 us. A fused
// version would need the cluster/DSMEM reduction inside the persistent loop.
#include <cuda_bf16.h>

#include <cstring>

#include "kernels.hpp"
#include "rownorm.cuh"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4, QD = 4, NORM_ROWS = 1, MAX_S = 4;
constexpr int kStageA = BM * BK * 2, kStageB = BN * BK * 2, kStage = kStageA + kStageB;   // 16 + 16 KB
constexpr int kChunkBytes = 32 * BM * 4;                 // 32 fp32 columns of a tile: 16 KB
constexpr int kStageBufBytes = 3 * kChunkBytes;           // up to S - 1 = 3 other partials of one chunk
constexpr int kSbuf = 2 * kStageBufBytes;                 // double-buffered (also holds an outgoing 64 KB tile)
constexpr int kSmem = STAGES * kStage + kSbuf + 512 + 1024;
constexpr int kTileFloats = BM * BN;

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// Debug trace (PB_CHAIN_TRACE=1; tools/chain_trace.py): per launch slot and item, globaltimer stamps of
// claim, activation dependency satisfied, accumulator ready, output published, plus smid / job / item.
constexpr int kTraceSlots = 64, kTraceItems = 1024;
constexpr size_t kTraceWords = (size_t)kTraceSlots * kTraceItems * 8;   // per table; two tables (items, chunks)
unsigned long long* g_trace_buf = nullptr;   // device buffer, allocated on the first traced launch
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#define TRACE(item, k, v)                                                                               \
    do {                                                                                                \
        if (a.trace_slot >= 0 && (item) < kTraceItems)                                                  \
            a.trace[((size_t)(a.trace_slot % kTraceSlots) * kTraceItems + (item)) * 8 + (k)] = (v);       \
    } while (0)

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// named barrier of the 4 epilogue warps (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ int job_per(const ChainJob& J) { return J.epi == EPI_SILU_MUL ? BN / 2 : BN; }
__device__ __forceinline__ int job_tiles(const ChainJob& J) { return (J.N + job_per(J) - 1) / job_per(J); }
__device__ __forceinline__ int job_items(const ChainArgs& a, const ChainJob& J) {
    return J.type == CHAIN_GEMM ? job_tiles(J) * J.S : (a.M_end - a.M_begin + NORM_ROWS - 1) / NORM_ROWS;
}
__device__ __forceinline__ int job_units(const ChainArgs& a, const ChainJob& J) {
    return J.type == CHAIN_GEMM ? job_tiles(J) : job_items(a, J);
}

// Spin until job j has published all its units, then acquire and order later TMA reads after it. The spin uses
// relaxed loads: an acquire load per iteration would invalidate the SM's L1 (CCTL.IVALL) every few hundred
// nanoseconds and stall the memory pipeline of every warp on the SM (measured: 4-5x slower epilogues).
__device__ __forceinline__ void wait_job(const ChainArgs& a, int j) {
    const uint32_t need = (uint32_t)job_units(a, a.job[j]);
    const uint32_t* p = a.ctl + 2 + j;
    uint64_t t0 = 0;
    unsigned ns = 64;
    while (ld_relaxed(p) < need) {
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (!t0) t0 = t;
        else if (t - t0 > 4000000000ull) __trap();   // 4 s: a broken dependency fails loudly instead of hanging
    }
    fence_acq_rel();
    fence_proxy_async_global();
}

// One norm row by the 4 epilogue warps, bit-identical to norm_kernel's 256-thread CTA (rownorm.cuh): thread et
// plays virtual threads et and et + 128 (virtual warps w and w + 4). PER_REG > 0: the row, gamma and beta are
// loaded into registers with every load in flight at once (d <= PER_REG * 256); 0: re-read per pass.
template <int PER_REG>
__device__ __forceinline__ void norm_row(const ChainJob& J, int r, int et, int lane, float* red) {
    const float* x = J.h + (size_t)r * J.ldh;
    const int d = J.d, per = (d + rownorm::kVT - 1) / rownorm::kVT, w = et >> 5;
    constexpr int NR = PER_REG > 0 ? PER_REG : 1;
    const bool has_beta = J.beta != nullptr;
    float v[NR][2], gm[NR][2], bt[NR][2];
    if (PER_REG > 0) {
#pragma unroll
        for (int i = 0; i < NR; ++i)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = et + 128 * k + rownorm::kVT * i;
                const bool ok = c < d;
                v[i][k] = ok ? __ldcg(x + c) : 0.f;
                gm[i][k] = ok ? __bfloat162float(J.gamma[c]) : 0.f;
                bt[i][k] = ok && has_beta ? __bfloat162float(J.beta[c]) : 0.f;
            }
    }
    auto val = [&](int i, int k) -> float {
        if (PER_REG > 0) return v[i][k];
        return __ldcg(x + et + 128 * k + rownorm::kVT * i);
    };
    const int n_i = PER_REG > 0 ? PER_REG : per;
    float mean = 0.f;
    if (has_beta) {
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int i = 0; i < n_i; ++i) {
            const int c = et + rownorm::kVT * i;
            if (c < d) s0 = rownorm::acc_sum(s0, val(i, 0));
            if (c + 128 < d) s1 = rownorm::acc_sum(s1, val(i, 1));
        }
        s0 = rownorm::warp_sum(s0);
        s1 = rownorm::warp_sum(s1);
        if (lane == 0) {
            red[w] = s0;
            red[w + 4] = s1;
        }
        epi_sync();
        mean = rownorm::mean_of(rownorm::combine8(red, lane), d);
        epi_sync();
    }
    float q0 = 0.f, q1 = 0.f;
#pragma unroll
    for (int i = 0; i < n_i; ++i) {
        const int c = et + rownorm::kVT * i;
        if (c < d) q0 = rownorm::acc_sq(q0, val(i, 0), mean);
        if (c + 128 < d) q1 = rownorm::acc_sq(q1, val(i, 1), mean);
    }
    q0 = rownorm::warp_sum(q0);
    q1 = rownorm::warp_sum(q1);
    if (lane == 0) {
        red[w] = q0;
        red[w + 4] = q1;
    }
    epi_sync();
    const float rstd = rownorm::rstd_of(rownorm::combine8(red, lane), d, J.eps);
    epi_sync();
    __nv_bfloat16* o = J.nout + (size_t)r * J.ldno;
#pragma unroll
    for (int i = 0; i < n_i; ++i)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int c = et + 128 * k + rownorm::kVT * i;
            if (c >= d) continue;
            if (PER_REG > 0)
                o[c] = rownorm::out_f(v[i][k], mean, rstd, gm[i][k], bt[i][k], has_beta);
            else
                o[c] = rownorm::out(val(i, k), mean, rstd, J.gamma, J.beta, c);
        }
}

__global__ void __launch_bounds__(192, 1) chain_kernel(const __grid_constant__ ChainArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sbuf = smem + STAGES * kStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(sbuf + kSbuf);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;   // [2] MMA -> epilogue
    uint64_t* acc_empty = acc_full + 2;    // [2] epilogue -> MMA (128 arrivals)
    uint64_t* q_full = acc_empty + 2;      // [QD] producer -> MMA + epilogue
    uint64_t* q_empty = q_full + QD;       // [QD] MMA (1) + epilogue warps (4) -> producer
    volatile int* qbuf = reinterpret_cast<volatile int*>(q_empty + QD);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(const_cast<int*>(qbuf + QD));
    float* red = reinterpret_cast<float*>(tmem_slot + 4);          // [8] norm group sums
    volatile int* last_flag = reinterpret_cast<volatile int*>(red + 8);
    uint64_t* rbar = reinterpret_cast<uint64_t*>(red + 16);        // [2] staging buffers filled (bulk loads)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int total = 0;
    for (int j = 0; j < a.n_jobs; ++j) total += job_items(a, a.job[j]);

    pdl_launch_dependents();
    if (tid == 0) {
        for (int j = 0; j < a.n_jobs; ++j)
            if (a.job[j].type == CHAIN_GEMM) {
                tma_prefetch_desc(&a.job[j].mx);
                tma_prefetch_desc(&a.job[j].mw);
            }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        for (int q = 0; q < QD; ++q) {
            mbar_init(&q_full[q], 1);
            mbar_init(&q_empty[q], 5);
        }
        mbar_init(&rbar[0], 1);
        mbar_init(&rbar[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<2 * BN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto decode = [&](int item, int& li) {
        int j = 0;
        for (; j < a.n_jobs; ++j) {
            const int n = job_items(a, a.job[j]);
            if (item < n) break;
            item -= n;
        }
        li = item;
        return j;
    };

    if (warp == 0) {
        if (lane == 0) {   // ---------------- producer: claim items, stream W early, X after the dependency
            int it = 0, qi = 0;
            bool waited = false;
            for (;;) {
                int item = (int)atomicAdd(a.ctl, 1u);
                if (item >= total) item = -1;
                const int slot = qi % QD;
                if (qi >= QD) mbar_wait(&q_empty[slot], ((qi / QD) - 1) & 1);
                qbuf[slot] = item;
                mbar_arrive(&q_full[slot]);
                ++qi;
                if (item < 0) break;
                TRACE(item, 0, gtime());
                int li;
                const int j = decode(item, li);
                TRACE(item, 5, ((unsigned long long)smid() << 48) | ((unsigned long long)j << 40) | (unsigned)li);
                const ChainJob& J = a.job[j];
                if (J.type != CHAIN_GEMM) continue;
                const int tile = li / J.S, split = li % J.S;
                const int n0 = tile * job_per(J);
                const int nk = (J.K + BK - 1) / BK;
                const int kb0 = (int)((long)nk * split / J.S), kb1 = (int)((long)nk * (split + 1) / J.S);
                const int my_k = kb1 - kb0, pre = my_k < STAGES ? my_k : STAGES;
                auto load_w = [&](int s, int kb) {
                    uint8_t* sB = smem + s * kStage + kStageA;
                    if (J.epi == EPI_SILU_MUL) {
                        tma_load_2d(sB, &J.mw, &full[s], kb * BK, n0);
                        tma_load_2d(sB + kStageB / 2, &J.mw, &full[s], kb * BK, J.up_row0 + n0);
                    } else {
                        tma_load_2d(sB, &J.mw, &full[s], kb * BK, n0);
                    }
                };
                for (int i = 0; i < pre; ++i) {   // weights: independent of every earlier job
                    const int g = it + i, s = g % STAGES;
                    if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], kStage);
                    load_w(s, kb0 + i);
                }
                if (j == 0) {
                    if (!waited) pdl_wait();   // job 0 reads the previous kernel's output
                    waited = true;
                } else {
                    wait_job(a, j - 1);
                }
                TRACE(item, 1, gtime());
                for (int i = 0; i < pre; ++i) {
                    const int s = (it + i) % STAGES;
                    tma_load_2d(smem + s * kStage, &J.mx, &full[s], (kb0 + i) * BK, a.M_begin);
                }
                for (int i = pre; i < my_k; ++i) {
                    const int g = it + i, s = g % STAGES;
                    mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], kStage);
                    tma_load_2d(smem + s * kStage, &J.mx, &full[s], (kb0 + i) * BK, a.M_begin);
                    load_w(s, kb0 + i);
                }
                it += my_k;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer (same instruction sequence as gemm_kernel per split)
            constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 0);
            int it = 0, qi = 0, g = 0;
            for (;;) {
                const int slot = qi % QD;
                mbar_wait(&q_full[slot], (qi / QD) & 1);
                const int item = qbuf[slot];
                mbar_arrive(&q_empty[slot]);
                ++qi;
                if (item < 0) break;
                int li;
                const ChainJob& J = a.job[decode(item, li)];
                if (J.type != CHAIN_GEMM) continue;
                const int split = li % J.S, nk = (J.K + BK - 1) / BK;
                const int my_k = (int)((long)nk * (split + 1) / J.S) - (int)((long)nk * split / J.S);
                const int b = g & 1;
                if (g >= 2) mbar_wait(&acc_empty[b], ((g >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t acc = tmem + b * BN;
                for (int i = 0; i < my_k; ++i, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(smem + s * kStage), b_base = a_base + kStageA;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(acc, smem_desc(a_base + k * 32, 16, 1024, kSw128),
                                  smem_desc(b_base + k * 32, 16, 1024, kSw128), idesc, (i | k) != 0 ? 1u : 0u);
                    umma_commit(&empty[s]);
                }
                umma_commit(&acc_full[b]);
                ++g;
            }
        }
    } else {   // ---------------- warps 2..5: GEMM epilogues (row = TMEM lane) and norm items
        const int et = tid - 64, quad = warp & 3, row_in_tile = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        pdl_wait();   // h / outputs of earlier kernels are read below
        int qi = 0, g = 0, red_uses = 0;
        for (;;) {
            const int slot = qi % QD;
            mbar_wait(&q_full[slot], (qi / QD) & 1);
            const int item = qbuf[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&q_empty[slot]);
            ++qi;
            if (item < 0) break;
            int li;
            const int j = decode(item, li);
            const ChainJob& J = a.job[j];
            if (J.type == CHAIN_NORM) {
                // ---- rows [r_a, r_b), each by all four epilogue warps
                if (et == 0) wait_job(a, j - 1);
                if (et == 0) TRACE(item, 1, gtime());
                epi_sync();
                const int r_a = a.M_begin + li * NORM_ROWS;
                const int r_b = min(a.M_end, r_a + NORM_ROWS);
                for (int r = r_a; r < r_b; ++r) {
                    if (J.d <= 8 * rownorm::kVT) norm_row<8>(J, r, et, lane, red);
                    else norm_row<0>(J, r, et, lane, red);
                }
                fence_proxy_async_global();   // x is read by the next job's TMA
                epi_sync();
                if (et == 0) red_release(a.ctl + 2 + j, 1);
                if (et == 0) TRACE(item, 4, gtime());
                continue;
            }
            // ---- GEMM item (tile, split)
            const int tile = li / J.S, split = li % J.S;
            const int b = g & 1;
            mbar_wait(&acc_full[b], (g >> 1) & 1);
            tc_fence_after();
            if (et == 0) TRACE(item, 2, gtime());
            const uint32_t acc = tmem + b * BN + lane_off;
            bool finish = true;
            if (J.S > 1) {
                // stage this split's fp32 tile in shared memory ([col/4][row] float4: conflict-free), one bulk
                // store to the workspace, then count the arrival; the last split of the tile finishes it
#pragma unroll 1
                for (int cb = 0; cb < BN / 32; ++cb) {
                    uint32_t r[32];
                    tmem_ld32_async(acc + cb * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<float4*>(sbuf)[(cb * 8 + q) * BM + row_in_tile] =
                            make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                }
                fence_proxy_async_smem();
                epi_sync();
                if (et == 0) {
                    bulk_store(a.part + ((size_t)tile * J.S + split) * kTileFloats, sbuf, kTileFloats * 4);
                    tma_store_commit();
                    tma_store_wait_all();
                    fence_proxy_async_global();
                    uint32_t* ctr = a.ctl + 8 + j * kChainMaxTiles + tile;
                    const bool last = atom_add_acq_rel(ctr, 1) == (uint32_t)J.S - 1;
                    if (last) {
                        *ctr = 0;   // every split of this tile has arrived: reset for the next launch
                        fence_proxy_async_global();
                    }
                    *last_flag = last;
                }
                epi_sync();
                finish = *last_flag != 0;
                if (et == 0) TRACE(item, 4, gtime());
            }
            if (finish) {
                const int n0 = tile * job_per(J);
                const int row = a.M_begin + row_in_tile;
                const bool row_ok = row < a.M_end;
                // 32-column chunks in the order they are consumed (SiLU: gate c with up c + 2)
                const bool silu_t = J.epi == EPI_SILU_MUL;
                auto chunk_of = [&](int k) { return silu_t ? ((k & 1) ? 2 + (k >> 1) : (k >> 1)) : k; };
                const int others = J.S - 1;
                // chunk k of the S - 1 other partials -> staging buffer k & 1 (others x 16 KB)
                auto issue = [&](int k) {
                    const int c = chunk_of(k);
                    uint64_t* bar = &rbar[k & 1];
                    mbar_arrive_expect_tx(bar, (uint32_t)others * kChunkBytes);
                    for (int s2 = 0, o = 0; s2 < J.S; ++s2) {
                        if (s2 == split) continue;
                        bulk_load(sbuf + (k & 1) * kStageBufBytes + o * kChunkBytes,
                                  reinterpret_cast<const uint8_t*>(a.part + ((size_t)tile * J.S + s2) * kTileFloats) +
                                      (size_t)c * kChunkBytes,
                                  kChunkBytes, bar);
                        ++o;
                    }
                };
                if (J.S > 1 && et == 0) {
                    issue(0);
                    issue(1);
                }
                // the fixed-order sum over splits 0..S-1 of chunk k (own split from TMEM)
                auto reduce32 = [&](int k, float (&v)[32]) {
                    uint32_t r[32];
                    tmem_ld32_async(acc + chunk_of(k) * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
                    if (J.S == 1) return;
                    mbar_wait(&rbar[k & 1], (uint32_t)((red_uses * 2 + (k >> 1)) & 1));
                    if (k == 0 && et == 0) TRACE(item, 6, gtime());
                    if (et == 0 && a.trace_slot >= 0 && item < kTraceItems)
                        a.trace[kTraceWords + ((size_t)(a.trace_slot % kTraceSlots) * kTraceItems + item) * 8 + 2 * k] =
                            gtime();
                    const float4* buf = reinterpret_cast<const float4*>(sbuf + (k & 1) * kStageBufBytes);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 s4;
#pragma unroll
                        for (int s2 = 0; s2 < MAX_S; ++s2) {
                            if (s2 >= J.S) break;
                            const int o = s2 < split ? s2 : s2 - 1;
                            const float4 p = s2 == split ? make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3])
                                                         : buf[o * (kChunkBytes / 16) + q * BM + row_in_tile];
                            if (s2 == 0) {
                                s4 = p;
                            } else {
                                s4.x += p.x;
                                s4.y += p.y;
                                s4.z += p.z;
                                s4.w += p.w;
                            }
                        }
                        v[4 * q] = s4.x;
                        v[4 * q + 1] = s4.y;
                        v[4 * q + 2] = s4.z;
                        v[4 * q + 3] = s4.w;
                    }
                };
                // after chunk(s) of staging buffer(s) have been read by every thread: refill them
                auto refill = [&](int k_done_lo, int k_done_hi) {
                    if (J.S == 1) return;
                    epi_sync();
                    if (et == 0)
                        for (int k = k_done_lo; k <= k_done_hi; ++k)
                            if (k + 2 < 4) issue(k + 2);
                };
                if (silu_t) {
#pragma unroll 1
                    for (int cb = 0; cb < 2; ++cb) {   // 32 gate columns + the matching 32 up columns
                        float gv[32], uv[32];
                        reduce32(2 * cb, gv);
                        reduce32(2 * cb + 1, uv);
                        refill(2 * cb, 2 * cb + 1);
                        const int n = n0 + cb * 32;
                        if (!row_ok || n >= J.N) continue;
                        __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(J.out) + (size_t)row * J.ldo + n;
#pragma unroll
                        for (int e = 0; e < 32; e += 2) {
                            const float o0 = silu(gv[e]) * uv[e], o1 = silu(gv[e + 1]) * uv[e + 1];
                            if (n + e + 1 < J.N) {
                                *reinterpret_cast<uint32_t*>(out + e) = bf16x2_bits(o0, o1);
                            } else if (n + e < J.N) {
                                out[e] = __float2bfloat16_rn(o0);
                            }
                        }
                    }
                } else {
#pragma unroll 1
                    for (int cb = 0; cb < BN / 32; ++cb) {
                        const int n = n0 + cb * 32;
                        const int nv = min(32, J.N - n);
                        float* hp = reinterpret_cast<float*>(J.out) + (size_t)row * J.ldo + n;
                        float4 hv[8];
                        const bool full32 = row_ok && nv == 32;
                        if (J.epi == EPI_RESID && full32) {   // residual loads in flight during the reduction
#pragma unroll
                            for (int q = 0; q < 8; ++q) hv[q] = __ldcg(reinterpret_cast<const float4*>(hp) + q);
                        }
                        float v[32];
                        reduce32(cb, v);
                        refill(cb, cb);
                        if (et == 0 && a.trace_slot >= 0 && item < kTraceItems)
                            a.trace[kTraceWords + ((size_t)(a.trace_slot % kTraceSlots) * kTraceItems + item) * 8 +
                                    2 * cb + 1] = gtime();
                        if (!row_ok || n >= J.N) continue;
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (J.bias && e < nv) v[e] += __bfloat162float(J.bias[n + e]);
                        if (J.epi == EPI_BF16) {
#pragma unroll
                            for (int e = 0; e < 32; ++e) {
                                if (n + e < J.scale_cols) v[e] *= J.scale;
                                if (J.relu) v[e] = fmaxf(v[e], 0.0f);
                            }
                            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(J.out) + (size_t)row * J.ldo + n;
                            if (nv == 32) {
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    *reinterpret_cast<uint4*>(out + 8 * q) = make_uint4(
                                        bf16x2_bits(v[8 * q], v[8 * q + 1]), bf16x2_bits(v[8 * q + 2], v[8 * q + 3]),
                                        bf16x2_bits(v[8 * q + 4], v[8 * q + 5]), bf16x2_bits(v[8 * q + 6], v[8 * q + 7]));
                            } else {
                                for (int e = 0; e < nv; ++e) out[e] = __float2bfloat16_rn(v[e]);
                            }
                        } else {   // EPI_RESID: h += acc + bias
                            if (full32) {
#pragma unroll
                                for (int q = 0; q < 8; ++q) {
                                    float4 x = hv[q];
                                    x.x += v[4 * q];
                                    x.y += v[4 * q + 1];
                                    x.z += v[4 * q + 2];
                                    x.w += v[4 * q + 3];
                                    reinterpret_cast<float4*>(hp)[q] = x;
                                }
                            } else {
                                for (int e = 0; e < nv; ++e) hp[e] = __ldcg(hp + e) + v[e];
                            }
                        }
                    }
                }
                if (J.S > 1) ++red_uses;
                if (et == 0) TRACE(item, 7, gtime());
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[b]);
            ++g;
            if (finish) {
                fence_proxy_async_global();   // outputs may be read by the next job's TMA
                epi_sync();
                if (et == 0) red_release(a.ctl + 2 + j, 1);
            }
            if (et == 0) TRACE(item, 3, gtime() | (finish ? 1ull << 63 : 0));
        }
    }

    // ---------------- teardown; the last CTA out re-zeroes the control words for the next use of this set
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<2 * BN>(tmem);
    }
    if (tid == 0) {
        if (atom_add_acq_rel(a.ctl + 1, 1) == gridDim.x - 1) {
            a.ctl[0] = 0;
            for (int j = 0; j < a.n_jobs; ++j) a.ctl[2 + j] = 0;
            a.ctl[1] = 0;
            __threadfence();
        }
    }
}

}  // namespace

int chain_norm_ok(int d) { return d >= 1 && d <= rownorm::kVT * 40 ? 1 : 0; }

size_t chain_part_bytes(int N, int K, int epi) {
    const int S = gemm_split_k(N, K, epi, BM);
    if (S <= 1) return 0;
    const int per = epi == EPI_SILU_MUL ? BN / 2 : BN;
    return (size_t)S * ((N + per - 1) / per) * kTileFloats * sizeof(float);
}

// Copy the trace of launch slots [0, n) to host memory (n * kTraceItems * 8 words), then the per-chunk trace.
cudaError_t chain_trace_copy(unsigned long long* host, int n) {
    if (n > kTraceSlots) n = kTraceSlots;
    const size_t words = (size_t)n * kTraceItems * 8;
    if (!g_trace_buf) {   // nothing traced yet
        memset(host, 0, 2 * words * sizeof(unsigned long long));
        return cudaSuccess;
    }
    cudaError_t e = cudaMemcpy(host, g_trace_buf, words * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    return cudaMemcpy(host + words, g_trace_buf + kTraceWords, words * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}

cudaError_t warm_chain_kernel() {
    cudaFuncAttributes at;
    return cudaFuncGetAttributes(&at, chain_kernel);
}

cudaError_t launch_chain(const ChainArgs& a, cudaStream_t s) {
    if (a.M_end <= a.M_begin || a.n_jobs <= 0) return cudaSuccess;
    if (a.M_end - a.M_begin > BM || a.n_jobs > kChainMaxJobs || !a.ctl) return cudaErrorInvalidValue;
    for (int j = 0; j < a.n_jobs; ++j) {
        const ChainJob& J = a.job[j];
        if (J.type == CHAIN_GEMM) {
            const int per = J.epi == EPI_SILU_MUL ? BN / 2 : BN;
            if (J.K <= 0 || J.K % 8 || J.S < 1 || J.S > MAX_S || (J.N + per - 1) / per > kChainMaxTiles) return cudaErrorInvalidValue;
            if (J.S > 1 && !a.part) return cudaErrorInvalidValue;
        } else if (!chain_norm_ok(J.d) || j == 0) {
            return cudaErrorInvalidValue;   // a norm item waits on the job before it
        }
    }
    cudaError_t e = smem_attr_once<chain_kernel>(kSmem);
    if (e != cudaSuccess) return e;
    ChainArgs args = a;
    if (args.trace_slot >= 0) {
        if (!g_trace_buf) {
            if ((e = cudaMalloc(&g_trace_buf, 2 * kTraceWords * sizeof(unsigned long long))) != cudaSuccess) return e;
            if ((e = cudaMemset(g_trace_buf, 0, 2 * kTraceWords * sizeof(unsigned long long))) != cudaSuccess) return e;
        }
        args.trace = g_trace_buf;
    }
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    }
    return launch_pdl(chain_kernel, dim3(sms), dim3(192), kSmem, s, a.pdl != 0, args);
}

}  // namespace pb
