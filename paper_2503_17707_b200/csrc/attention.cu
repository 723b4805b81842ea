// attention.cu — causal prefill attention on the tensor cores (tcgen05 / TMEM / TMA), head dim 64 or 128.
//
//   a_t = sum_{j <= t} softmax_j(q_t . k_j * score_scale) v_j        (per head; GQA: kv head = h / group)
//   (the attention of every decoder layer in the first-token prefill; HF conventions G14)
//
// CTA = (128 query positions, head, sequence); 288 threads:
//   warps 0-7 : softmax + epilogue, two threads per query row (TMEM lane): warp q and warp q + 4 take key columns
//               [0, 64) and [64, 128) of each S tile (2 softmax warps per SMSP hide each other's stalls)
//   warp 8    : TMA producer and single-thread MMA issuer
// Two passes over the 128-key tiles j (keys [0, q_tile_end) only — causal), so that the probabilities are rounded
// to bf16 after normalisation, at exactly the storage contract's rounding point:
//   pass A:  S = Q K_j^T   tcgen05.mma M128 N128, K = hd, fp32 accumulator in TMEM columns [0, 128);
//            softmax threads: tcgen05.ld the row, mask j > t, running max m (exact) and l = sum exp2(s*c - m)
//   pass B:  S = Q K_j^T again; P = RNE_bf16(exp2(s*c - m) / l) stored as bf16 pairs into TMEM (tcgen05.st);
//            O += P V_j    tcgen05.mma M128 N=hd, K = 128 keys, A = P read from TMEM, V read MN-major straight
//                          from its TMA tile, fp32 accumulator in TMEM columns [128, 128 + hd)
//   out = RNE_bf16(O)
// K streams through a 2-buffer ring over the 2 x n_kv iterations (K of iteration i+2 loads while softmax i runs),
// V is double-buffered in pass B; S_{i+1} is issued as soon as softmax i has read S_i. Q/K/V come through one
// 3-D tensor map over the token-major qkv rows (col, sequence b, position t) whose t extent is t1, so keys
// past the last computed position are zero-filled by TMA, never read.
// Cost of contract-exact rounding: the QK^T MMAs and the exponentials run twice (pass A has no PV).
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdlib>

#include "kernels.hpp"
#include "sm100.cuh"

namespace pb {
using namespace sm100;

namespace {

constexpr int QT = 128, KT = 128;
constexpr int kAtom = 128 * 128;       // one 128-row x 64-col bf16 SW128 box = 16 KB

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Sums of exp2 over a thread's scores run in 8 independent chains combined in a fixed tree (deterministic); the
// row max likewise (exact in any order).
__device__ __forceinline__ float tree8(const float (&r)[8]) {
    return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

// TWO = false: one CTA per SM, K and V double-buffered, P in its own TMEM columns (S 128 | O HD | P 64 -> 512).
// TWO = true : two CTAs per SM (the other CTA's work hides this one's load and handshake latency): K and V single-
//              buffered (Q + K + V = 96 KB at hd 128), P written over the S columns it came from (S/P 128 | O HD
//              -> 256 TMEM columns per CTA), so S_{i+1} of pass B waits for PV_i.
template <int HD, bool TWO>
struct AttnSmem {
    static constexpr int kQ = HD / 64 * kAtom, kK = kQ, kV = kQ;
    static constexpr int NBUF = TWO ? 1 : 2;
    static constexpr int offQ = 0, offK = offQ + kQ, offV = offK + NBUF * kK, offBar = offV + NBUF * kV;
    static constexpr int offX = offBar + 128;   // half-row exchange: [2 halves][128 rows] float
    static constexpr uint32_t kTmemCols = TWO || HD == 64 ? 256 : 512;
    static constexpr int kTotal = offX + 2 * 128 * 4 + 1024;
};

template <int HD, bool TWO>
__global__ void __launch_bounds__(288, TWO ? 2 : 1) attention_tc_kernel(const __grid_constant__ CUtensorMap map, __nv_bfloat16* __restrict__ out,
                                                        int ldo, int t0, int t1, int group, int k_col0, int v_col0,
                                                        float scale_log2, const int* dyn, int seq_stride) {
    using SM = AttnSmem<HD, TWO>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem + SM::offQ, *sK = smem + SM::offK, *sV = smem + SM::offV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::offBar);
    uint64_t *q_full = bars, *k_full = bars + 1 /* [2] */, *v_full = bars + 3 /* [2] */, *s_full = bars + 5,
             *s_free = bars + 6, *p_full = bars + 7, *o_full = bars + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
    float* xch = reinterpret_cast<float*>(smem + SM::offX);   // [half][row]

    pdl_launch_dependents();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // grid (head, sequence, query tile): the block scheduler hands out CTAs with x fastest, so every head's and
    // sequence's LATEST query tile (the most key tiles) starts first and the one-tile CTAs fill the tail (longest
    // processing time first; with (tile, head) order the last wave was a few long CTAs on otherwise idle SMs)
    const int h = blockIdx.x, b = blockIdx.y, kvh = h / group;
    if (dyn) {   // f3 decode graph: the position is read on the device
        t0 += *dyn;
        t1 += *dyn;
    }
    const int qtile = gridDim.z - 1 - blockIdx.z;          // longest (latest) query tiles first
    const int q0 = t0 + qtile * QT;
    const int q_hi = min(q0 + QT, t1);
    const int n_kv = (q_hi + KT - 1) / KT;                  // key tiles [0, n_kv)

    if (tid == 0) {
        tma_prefetch_desc(&map);
        mbar_init(q_full, 1);
        mbar_init(&k_full[0], 1);
        mbar_init(&k_full[1], 1);
        mbar_init(&v_full[0], 1);
        mbar_init(&v_full[1], 1);
        mbar_init(s_full, 1);
        mbar_init(s_free, 8);      // one arrive per softmax warp
        mbar_init(p_full, 8);
        mbar_init(o_full, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<SM::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tO = tmem + 128, tP = TWO ? tmem : tmem + 128 + HD;
    // packed P of key half hf (keys hf*64 .. hf*64+63, 32 columns) starts at tP + hf * kPHalf: with P written over S
    // (TWO) each half writes into ITS OWN S columns [hf*64, hf*64+32), never into columns its partner thread may
    // not have read yet
    constexpr uint32_t kPHalf = TWO ? 64 : 32;
    pdl_wait();   // q/k/v are the previous kernel's output

    // Two passes over the key tiles, so the probabilities are rounded to bf16 AFTER normalisation, exactly where the
    // storage contract rounds them (P = RNE_bf16(softmax(S))):
    //   pass A (iterations i < n_kv):  S_j -> row max m and row sum l = sum exp2(s*c - m) (exact rescale per tile)
    //   pass B (iterations i >= n_kv): S_j again -> P = RNE_bf16(exp2(s*c - m) / l) -> O += P V_j
    // The output is then RNE_bf16(O) with no final division.
    // One key tile (T <= 128: C2's prompt, short decode contexts): the row max and sum come from the same S the
    // probabilities use, so a single pass computes E = exp2(s*c - m) once, l = sum E, P = RNE_bf16(E / l) — the same
    // values, in the same order, as the two passes would (no second QK^T, no second exponential).
    const bool single = n_kv == 1;
    const int NI = single ? 1 : 2 * n_kv;
    if (warp == 8) {
        if (lane == 0) {
            constexpr int kBox = kAtom;   // bytes of one 64-col box
            auto load_rows = [&](uint8_t* dst, uint64_t* bar, int col, int t) {
#pragma unroll
                for (int a = 0; a < HD / 64; ++a) {
                    if (seq_stride) tma_load_3d(dst + a * kBox, &map, bar, col + a * 64, t, b);   // (col, t, b)
                    else tma_load_3d(dst + a * kBox, &map, bar, col + a * 64, b, t);              // (col, b, t)
                }
            };
            auto kv_of = [&](int i) { return single ? 0 : (i < n_kv ? i : i - n_kv); };
            mbar_arrive_expect_tx(q_full, SM::kQ);
            load_rows(sQ, q_full, h * HD, q0);
            constexpr int NB = SM::NBUF;
            for (int i = 0; i < NB && i < NI; ++i) {   // K of the first iteration(s)
                mbar_arrive_expect_tx(&k_full[i], SM::kK);
                load_rows(sK + i * SM::kK, &k_full[i], k_col0 + kvh * HD, kv_of(i) * KT);
            }
            for (int j = 0; j < NB && j < n_kv; ++j) {   // V of the first pass-B iteration(s)
                mbar_arrive_expect_tx(&v_full[j], SM::kV);
                load_rows(sV + j * SM::kV, &v_full[j], v_col0 + kvh * HD, j * KT);
            }
            constexpr uint32_t idS = idesc_bf16_f32(128, 128, 0, 0);
            constexpr uint32_t idO = idesc_bf16_f32(128, HD, 0, 1);
            mbar_wait(q_full, 0);
            auto issue_S = [&](int i) {   // S = Q K^T into the (single) S columns
                const int kb = i % NB;
                mbar_wait(&k_full[kb], (i / NB) & 1);
                tc_fence_after();
                const uint32_t kbase = smem_u32(sK + kb * SM::kK);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                    umma_bf16(tS, smem_desc(smem_u32(sQ) + off, 16, 1024, kSw128),
                              smem_desc(kbase + off, 16, 1024, kSw128), idS, kk > 0 ? 1u : 0u);
                }
                umma_commit(s_full);
            };
            issue_S(0);
            for (int i = 0; i < NI; ++i) {
                const uint32_t ph = i & 1;
                // ---- S_i done: its K buffer takes the K of iteration i + NB
                mbar_wait(s_full, ph);
                if (i + NB < NI) {
                    const int kb = i % NB;
                    mbar_arrive_expect_tx(&k_full[kb], SM::kK);
                    load_rows(sK + kb * SM::kK, &k_full[kb], k_col0 + kvh * HD, kv_of(i + NB) * KT);
                }
                const bool pass_a = i < n_kv && !single;
                // ---- S_{i+1} as soon as the softmax has read S_i out of TMEM (pass A, or P in its own columns)
                if (i + 1 < NI) {
                    mbar_wait(s_free, ph);
                    if (pass_a || !TWO) issue_S(i + 1);
                }
                if (pass_a) continue;
                const int j = single ? 0 : i - n_kv;
                // ---- V_{j+NB} into the buffer PV_{j+NB-2} has finished reading (double-buffered V)
                if (!TWO && j >= 1 && j + 1 < n_kv) {
                    mbar_wait(o_full, (j - 1) & 1);
                    const int vb = (j + 1) & 1;
                    mbar_arrive_expect_tx(&v_full[vb], SM::kV);
                    load_rows(sV + vb * SM::kV, &v_full[vb], v_col0 + kvh * HD, (j + 1) * KT);
                }
                // ---- O += P_j V_j
                mbar_wait(p_full, j & 1);
                mbar_wait(&v_full[j % NB], (j / NB) & 1);
                tc_fence_after();
                const uint32_t vbase = smem_u32(sV + (j % NB) * SM::kV);
#pragma unroll
                for (int kk = 0; kk < KT / 16; ++kk) {
                    // A = P from TMEM: 16 keys = 8 packed columns. B = V tile [128 keys x hd], hd contiguous
                    // (MN-major): 64-col boxes kBox apart (LBO), 8-key groups 1024 B apart (SBO); 16 keys = 2048 B.
                    const uint64_t bd = smem_desc(vbase + kk * 2048, kBox, 1024, kSw128);
                    umma_bf16_ts(tO, tP + (kk >> 2) * kPHalf + (kk & 3) * 8, bd, idO, (j > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(o_full);
                if (TWO && i + 1 < NI) {   // P_j lives in S's columns and V_j in the only V buffer: both free after PV_j
                    mbar_wait(o_full, j & 1);
                    if (j + 1 < n_kv) {
                        mbar_arrive_expect_tx(&v_full[0], SM::kV);
                        load_rows(sV, &v_full[0], v_col0 + kvh * HD, (j + 1) * KT);
                    }
                    issue_S(i + 1);
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- softmax warps: TWO threads per query row r: warps q and q + 4 (TMEM lane quadrant q) hold
        // key columns [0, 64) and [64, 128) of every S tile — 8 softmax warps, 2 per SMSP, so one's dependency stalls
        // hide behind the other's issue. Per tile the halves exchange their row maxima (shared memory + a 64-thread
        // named barrier per quadrant); each keeps the running sum of its own half, combined once after pass A.
        const int q4 = warp & 3, hf = warp >> 2;
        const int r = q4 * 32 + lane;
        const int t = q0 + r;
        const bool row_ok = t < q_hi;   // rows past t1 are computed (never masked, always finite) but not stored
        const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
        const int bar_id = 1 + q4;      // named barrier of the two warps of quadrant q4
        auto pair_sync = [&]() { named_bar_sync(bar_id, 64); };
        auto exchange = [&](float v) {  // the partner half's value of this row
            xch[hf * 128 + r] = v;
            pair_sync();
            const float o = xch[(hf ^ 1) * 128 + r];
            pair_sync();                 // the slots are rewritten by the next exchange
            return o;
        };
        float m = -CUDART_INF_F, l = 0.f, inv_l = 0.f;
        for (int i = 0; i < NI; ++i) {
            const uint32_t ph = i & 1;
            const bool pass_b = single || i >= n_kv;
            const int j = single ? 0 : (pass_b ? i - n_kv : i);
            mbar_wait(s_full, ph);
            tc_fence_after();
            uint32_t sr[2][32];
#pragma unroll
            for (int c = 0; c < 2; ++c) tmem_ld32_async(tS + lane_off + hf * 64 + c * 32, sr[c]);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_free);
            // causal mask (key > t) only on the tiles that reach past the first query of this query tile
            const int key0 = j * KT + hf * 64;
            if (key0 + 63 > q0) {
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (key0 + c * 32 + e > t) sr[c][e] = __float_as_uint(-CUDART_INF_F);
            }
            auto half_max = [&]() {
                float mk[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) mk[k] = -CUDART_INF_F;
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) mk[e & 7] = fmaxf(mk[e & 7], __uint_as_float(sr[c][e]));
                return fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])),
                             fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
            };
            if (single) {   // ---- one key tile: max, E = exp2(s*c - m) kept in sr, l = sum E, P = E / l
                const float hm = half_max();
                m = fmaxf(hm, exchange(hm)) * scale_log2;
                float rk[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float ev = fast_exp2(fmaf(__uint_as_float(sr[c][e]), scale_log2, -m));
                        sr[c][e] = __float_as_uint(ev);
                        rk[e & 7] += ev;
                    }
                const float lh = tree8(rk);
                const float lo = exchange(lh);
                l = hf == 0 ? lh + lo : lo + lh;   // the same sum (half 0 first) in both threads
                inv_l = 1.f / l;
#pragma unroll
                for (int cb = 0; cb < 2; ++cb) {
                    uint32_t w[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        w[e] = bf16x2_bits(__uint_as_float(sr[cb][2 * e]) * inv_l,
                                           __uint_as_float(sr[cb][2 * e + 1]) * inv_l);
                    tmem_st16(tP + lane_off + hf * kPHalf + cb * 16, w);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full);
                continue;
            }
            if (!pass_b) {
                // ---- pass A: exact running max of the whole row (halves exchanged) and this half's rescaled sum
                const float hm = half_max();
                const float m_new = fmaxf(m, fmaxf(hm, exchange(hm)) * scale_log2);
                float rk[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) rk[e & 7] += fast_exp2(fmaf(__uint_as_float(sr[c][e]), scale_log2, -m_new));
                const float rs = tree8(rk);
                l = (m == -CUDART_INF_F ? 0.f : l * fast_exp2(m - m_new)) + rs;
                m = m_new;
                continue;
            }
            // ---- pass B: P = RNE_bf16(exp2(s*c - m) / l) straight into TMEM (the A operand of the PV MMA)
            if (j == 0) {   // the row sum: both halves' running sums at the final max (half 0 first)
                const float lo = exchange(l);
                l = hf == 0 ? l + lo : lo + l;
                inv_l = 1.f / l;   // l >= 1: the row maximum contributes exp2(0)
            }
            // the probabilities are computed (packed in place into sr[cb][0..15]) while PV_{j-1} still reads the
            // previous P from TMEM; only the stores wait for it
#pragma unroll
            for (int cb = 0; cb < 2; ++cb)
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float p0 = fast_exp2(fmaf(__uint_as_float(sr[cb][2 * e]), scale_log2, -m)) * inv_l;
                    const float p1 = fast_exp2(fmaf(__uint_as_float(sr[cb][2 * e + 1]), scale_log2, -m)) * inv_l;
                    sr[cb][e] = bf16x2_bits(p0, p1);
                }
            if (j > 0) {   // P (TMEM) is read by PV_{j-1}
                mbar_wait(o_full, (j - 1) & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int cb = 0; cb < 2; ++cb) {
                uint32_t w[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) w[e] = sr[cb][e];
                tmem_st16(tP + lane_off + hf * kPHalf + cb * 16, w);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
        }
        // ---------------- epilogue: out = RNE_bf16(O), each half of the row's HD columns by one of the two threads
        mbar_wait(o_full, (n_kv - 1) & 1);
        tc_fence_after();
        __nv_bfloat16* o_row =
            out + (seq_stride ? (size_t)b * seq_stride + t : (size_t)t * gridDim.y + b) * ldo + h * HD;
#pragma unroll
        for (int c = hf * (HD / 64); c < (hf + 1) * (HD / 64); ++c) {
            uint32_t o[32];
            tmem_ld32_async(tO + lane_off + c * 32, o);
            tmem_wait_ld();
            if (row_ok) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 w;
                    w.x = bf16x2_bits(__uint_as_float(o[8 * q + 0]), __uint_as_float(o[8 * q + 1]));
                    w.y = bf16x2_bits(__uint_as_float(o[8 * q + 2]), __uint_as_float(o[8 * q + 3]));
                    w.z = bf16x2_bits(__uint_as_float(o[8 * q + 4]), __uint_as_float(o[8 * q + 5]));
                    w.w = bf16x2_bits(__uint_as_float(o[8 * q + 6]), __uint_as_float(o[8 * q + 7]));
                    *reinterpret_cast<uint4*>(o_row + c * 32 + q * 8) = w;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc<SM::kTmemCols>(tmem);
    }
}

template <int HD, bool TWO>
cudaError_t launch_tc(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t0, int t1, int B, int H,
                      int group, int k_col0, int v_col0, float score_scale, cudaStream_t s, bool pdl,
                      const int* dyn, int t_extent, int seq_stride) {
    // 3-D view of the token-major rows: (col, sequence b, position t), t extent = t1 (keys >= t1 zero-filled);
    // a decode graph's positions are only known on the device: the view then spans t_extent positions and the
    // causal mask (key <= query) keeps later rows out.
    const uint64_t T_ext = (uint64_t)(dyn ? t_extent : t1);
    const uint64_t dims_tm[3] = {(uint64_t)ld, (uint64_t)B, T_ext}, dims_sm[3] = {(uint64_t)ld, T_ext, (uint64_t)B};
    const uint64_t str_tm[2] = {(uint64_t)ld * 2, (uint64_t)ld * 2 * B};
    const uint64_t str_sm[2] = {(uint64_t)ld * 2, (uint64_t)ld * 2 * (uint64_t)seq_stride};
    const uint32_t box_tm[3] = {64, 1, 128}, box_sm[3] = {64, 128, 1};
    const uint64_t* dims = seq_stride ? dims_sm : dims_tm;
    const uint64_t* strides = seq_stride ? str_sm : str_tm;
    const uint32_t* box = seq_stride ? box_sm : box_tm;
    CUtensorMap map;
    char err[256];
    if (!make_map_bf16_3d(&map, qkv, dims, strides, box, 128, err, sizeof err)) return cudaErrorInvalidValue;
    using SM = AttnSmem<HD, TWO>;
    cudaError_t e = smem_attr_once<attention_tc_kernel<HD, TWO>>(SM::kTotal);
    if (e != cudaSuccess) return e;
    const dim3 grid(H, B, (t1 - t0 + QT - 1) / QT);
    const float scale_log2 = score_scale * 1.4426950408889634f;
    return launch_pdl(attention_tc_kernel<HD, TWO>, grid, 288, SM::kTotal, s, pdl, map, out, ldo, t0, t1, group, k_col0,
                      v_col0, scale_log2, dyn, seq_stride);
}

// Longest context (keys) that takes the SIMT decode kernel (PB_DECODE_MAX_KEYS overrides, for measurement).
int kDecodeAttnMaxKeys() {
    static const int v = getenv("PB_DECODE_MAX_KEYS") ? atoi(getenv("PB_DECODE_MAX_KEYS")) : 12288;
    return v;
}

}  // namespace

cudaError_t warm_attention_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, attention_tc_kernel<64, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, attention_tc_kernel<128, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, attention_tc_kernel<64, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, attention_tc_kernel<128, true>);
    return e;
}

cudaError_t launch_attention(const __nv_bfloat16* qkv, int ld, __nv_bfloat16* out, int ldo, int t0, int t1, int B,
                             int n_heads, int n_kv_heads, int hd, int k_col0, int v_col0, float score_scale,
                             cudaStream_t s, bool pdl, const int* dyn, int t_extent, int seq_stride) {
    if (t1 <= t0) return cudaSuccess;
    const bool tma_ok = (ld % 8) == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 && (ldo % 8) == 0 &&
                        (k_col0 % 8) == 0 && (v_col0 % 8) == 0;
    const int group = n_heads / n_kv_heads;
    // one query position per sequence (decode steps): the SIMT decode kernel (a cluster of CTAs per head and
    // sequence splitting the keys; launch_decode_attention). Measured (profiles/r02_decode_attention_ab.txt): C2
    // decode 1.065 -> 1.009 ms per token, C4 6.80 -> 5.83 ms. The choice depends on the context bound (max_keys: the
    // decode graph's position range), not on the step's position.
    static const bool dec_off = getenv("PB_DECODE_ATTN") && atoi(getenv("PB_DECODE_ATTN")) == 0;   // A/B
    const int max_keys = dyn ? t_extent : t1;
    if (t1 - t0 == 1 && !seq_stride && !dec_off && (hd == 64 || hd == 128) && (ld % 8) == 0 && (k_col0 % 8) == 0 &&
        (v_col0 % 8) == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 && max_keys <= kDecodeAttnMaxKeys())
        return launch_decode_attention(qkv, ld, out, ldo, t1, B, n_heads, n_kv_heads, hd, k_col0, v_col0, score_scale,
                                       s, pdl, dyn, max_keys);
    static const bool two = !getenv("PB_ATTN_ONE") ;   // two CTAs per SM unless PB_ATTN_ONE (A/B measurement)
    if (tma_ok && hd == 64 && two)
        return launch_tc<64, true>(qkv, ld, out, ldo, t0, t1, B, n_heads, group, k_col0, v_col0, score_scale, s, pdl,
                                   dyn, t_extent, seq_stride);
    if (tma_ok && hd == 128 && two)
        return launch_tc<128, true>(qkv, ld, out, ldo, t0, t1, B, n_heads, group, k_col0, v_col0, score_scale, s, pdl,
                                    dyn, t_extent, seq_stride);
    if (tma_ok && hd == 64)
        return launch_tc<64, false>(qkv, ld, out, ldo, t0, t1, B, n_heads, group, k_col0, v_col0, score_scale, s, pdl, dyn,
                                    t_extent, seq_stride);
    if (tma_ok && hd == 128)
        return launch_tc<128, false>(qkv, ld, out, ldo, t0, t1, B, n_heads, group, k_col0, v_col0, score_scale, s, pdl, dyn,
                                     t_extent, seq_stride);
    if (dyn || seq_stride) return cudaErrorNotSupported;   // decode graphs / sequence-major: tensor-core kernel only
    return launch_attention_simt(qkv, ld, out, ldo, t0, t1, B, n_heads, n_kv_heads, hd, k_col0, v_col0, score_scale,
                                 s);
}

}  // namespace pb
