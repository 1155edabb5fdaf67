// gemm_tc.cu -- tcgen05 tensor-core GEMMs of a4/a6 for bf16 storage (fp32 accumulate in TMEM).
//
//   k_gemm_tc_nn : C[M x N] = [A1 | A2][M x K] * B           (feature transform, dH = dT W^T)
//   k_gemm_tc_tn : dW[K x N] = [A1 | A2]^T * Bm, split over row slabs (weight gradient)
//
// B200 design.  The transform is tall-skinny (M = 10^5..10^8 node rows, K, N <= 256) and
// HBM-bound (~64 FLOP/B), so the kernels are built to stream rows at full bandwidth:
//  * persistent CTAs (one per SM), warp-specialised: warp 0 = TMA producer, warp 1 = single-
//    thread tcgen05.mma issuer (+ TMEM owner), warps 2-5 = epilogue (TMEM -> regs -> smem);
//  * A tiles (128 rows x 64 bf16 = one 128-byte SWIZZLE_128B atom row per node) arrive by
//    TMA into a 4-stage mbarrier ring; OOB rows / columns are zero-filled by TMA;
//  * the weights (the whole K x N operand, <= 64 KB bf16) are converted fp32 -> bf16 once per
//    CTA into the K-major SW128 canonical layout and stay resident in shared memory;
//  * accumulators double-buffered in TMEM (2 x N columns) so the epilogue of tile i overlaps
//    the MMAs of tile i+1.  Fused epilogue: relu'-mask (mask tile TMA-loaded into smem by the
//    producer) or ReLU, bf16 cast, column split; the result tile is staged in SW128 smem and
//    written by TMA bulk-tensor stores (coalesced, asynchronous, clipped at the tensor edge).
//  * The weight gradient reads both operands MN-major straight from the row-major node
//    tensors (A = h_in^T, B = dZ^T as UMMA operands), accumulates a CTA's row slab in TMEM
//    and writes an fp32 partial; partials are summed in slab order (deterministic split-K).
#include <cudaTypedefs.h>

#include "gemm.cuh"
#include "tc.cuh"

namespace grappa {

constexpr int kTcThreads = 192;
constexpr int kNNThreads = 320;          // producer, MMA, 2 x 4 epilogue warps
constexpr int kMaxNNStages = 8;
constexpr int kNNStageBytes = 128 * 128;    // 128 rows x 128 B
constexpr int kBoxBytes = 128 * 128;        // one 64-column x 128-row bf16 SW128 box
constexpr int kTNMaxStages = 8;
constexpr int kMaxSmem = 227 * 1024;
// weight-gradient split plan: a fixed CTA budget (= B200 SM count) so workspace sizing and
// the slab partition (hence the summation order) do not depend on the device queried
constexpr int kTnCtas = 148;

struct TcNN {
    int64_t M;
    int K1, K2, N, kb1, kb2;
    const float* B;
    const float* rs;
    int b_trans;
    int relu;
    int has_mask;
    int n_split;
    int nb1, nb2;          // 64-column output boxes of C1 / C2
    int num_tiles;
    int stages;            // A-tile ring depth (<= kMaxNNStages)
    int mask_tma;          // relu'-gate boxes TMA-staged one tile ahead (else register prefetch)
    int nsb;               // staging boxes per epilogue group (1 or 2)
    uint32_t tmem_cols;
    // weights too large to stay resident (K x N bf16 > the shared memory left by the ring, e.g.
    // cora's K = 1440 input layer): the weight k-block travels with each A tile instead, from a
    // global image already in the SW128 K-major layout (k_weight_image), by a plain bulk copy
    int b_stream;
    const uint8_t* bimg;
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(tc::smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Stage the fp32 weights once per CTA as the bf16 B operand: [kb][N rows][64 k] K-major,
// SWIZZLE_128B, k >= K zero; W1 rows [0, K1) fill k-blocks [0, kb1), rows [K1, Kt) the rest.
// One thread per 16-byte chunk (operand row n, 8 consecutive k): consecutive threads take
// consecutive n, so the reads of W [Kt x N] are coalesced (b_trans: W stored [N x Kt], 32
// contiguous bytes per thread); 8 independent loads per chunk and 4 chunks unrolled keep the
// prologue short (it was a serial chain of dependent loads and 2-byte scattered stores).
// sBlo != nullptr also stages the residual lo = bf16(w - bf16(w)) (split-fp32 GEMMs).
__device__ __forceinline__ void stage_weights(uint8_t* sB, uint8_t* sBlo, const float* __restrict__ B, int K1,
                                              int K2, int N, int kb1, int kbt, int b_trans) {
    const int Kt = K1 + K2;
    const int total = kbt * 8 * N;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int n = idx % N, kc = idx / N;
        const int kb = kc >> 3, c8 = kc & 7;
        int k0, kend;
        if (kb < kb1) { k0 = kb * 64 + c8 * 8; kend = K1; }
        else { k0 = K1 + (kb - kb1) * 64 + c8 * 8; kend = Kt; }
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int k = k0 + j;
            v[j] = k < kend ? __ldg(b_trans ? B + (int64_t)n * Kt + k : B + (int64_t)k * N + n) : 0.f;
        }
        uint32_t h[4], l[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const __nv_bfloat162 bh = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            const float2 fh = __bfloat1622float2(bh);
            const __nv_bfloat162 bl = __floats2bfloat162_rn(v[2 * j] - fh.x, v[2 * j + 1] - fh.y);
            h[j] = *reinterpret_cast<const uint32_t*>(&bh);
            l[j] = *reinterpret_cast<const uint32_t*>(&bl);
        }
        const uint32_t off = (uint32_t)kb * N * 128 + tc::sw128_off(n, c8);
        *reinterpret_cast<uint4*>(sB + off) = make_uint4(h[0], h[1], h[2], h[3]);
        if (sBlo) *reinterpret_cast<uint4*>(sBlo + off) = make_uint4(l[0], l[1], l[2], l[3]);
    }
}

// the same bf16 K-major SWIZZLE_128B image stage_weights writes to shared memory, written to global
// memory once per call: k-block kb at byte kb * N * 128 (a multiple of 1024, so the swizzle of the
// image equals the swizzle of a 1024-aligned shared-memory copy of it)
__global__ void k_weight_image(const float* __restrict__ B, int K1, int K2, int N, int kb1, int kbt, int b_trans,
                               uint8_t* __restrict__ img) {
    const int Kt = K1 + K2;
    const int total = kbt * 8 * N;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int n = idx % N, kc = idx / N;
        const int kb = kc >> 3, c8 = kc & 7;
        int k0, kend;
        if (kb < kb1) { k0 = kb * 64 + c8 * 8; kend = K1; }
        else { k0 = K1 + (kb - kb1) * 64 + c8 * 8; kend = Kt; }
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int k = k0 + j;
            v[j] = k < kend ? __ldg(b_trans ? B + (int64_t)n * Kt + k : B + (int64_t)k * N + n) : 0.f;
        }
        uint32_t h[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const __nv_bfloat162 bh = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            h[j] = *reinterpret_cast<const uint32_t*>(&bh);
        }
        *reinterpret_cast<uint4*>(img + (size_t)kb * N * 128 + tc::sw128_off(n, c8)) = make_uint4(h[0], h[1], h[2], h[3]);
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(tc::smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void grp_bar(int h) { asm volatile("bar.sync %0, 128;" ::"r"(1 + h) : "memory"); }

// Epilogue of one tile for epilogue group H (4 warps = the 4 TMEM lane quarters).  The 64-column
// output boxes alternate between the two groups, so two groups drain one accumulator in
// parallel.  Each group stages its boxes in its own `nsb` SW128 buffers (TMA stores).
template <int H>
__device__ __forceinline__ void nn_epilogue(const TcNN& p, const CUtensorMap* tmC1, const CUtensorMap* tmC2,
                                            const __nv_bfloat16* __restrict__ mask, uint8_t* sbuf, int nsb,
                                            uint32_t tmem_acc, uint64_t* tfull, uint32_t aphase,
                                            int ew, int lane, int tile, bool leader, int& ob, float rsv,
                                            const uint8_t* gsm) {
    const int r = ew * 32 + lane;                 // row within the tile
    // relu'-mask of this thread's row for this group's C1 chunks (C1 chunk j lies in box j >> 2,
    // owned by group (j >> 2) & 1), fetched before waiting so the latency hides under the MMAs
    const int64_t grow = (int64_t)tile * 128 + r;
    const bool live = grow < p.M;
    const uint4* msrc = reinterpret_cast<const uint4*>(mask + (live ? grow : 0) * p.n_split);
    tc::mbar_wait(tfull, aphase);
    tc::fence_after();
    const uint32_t tbase = tmem_acc + ((uint32_t)(ew * 32) << 16);
    const int nbo = p.nb1 + p.nb2;
#pragma unroll 1
    for (int bx = H; bx < nbo; bx += 2) {
        const bool first = bx < p.nb1;
        const int cbase = first ? bx * 64 : (bx - p.nb1) * 64;              // column inside C1 / C2
        const int cend = first ? min(cbase + 64, p.n_split) : min(cbase + 64, p.N - p.n_split);
        const int coff = first ? 0 : p.n_split;                              // accumulator column
        uint8_t* obox = sbuf + (nsb == 2 ? (ob & 1) : 0) * kBoxBytes;
        if (leader) {
            if (nsb == 2) bulk_wait_read1();          // the store that last used this buffer is done
            else bulk_wait_read0();
        }
        grp_bar(H);
#pragma unroll
        for (int q2 = 0; q2 < 4; q2 += 2) {
            if (cbase + q2 * 16 >= cend) break;
            // two 16-column TMEM loads in flight per wait
            uint32_t raw[2][16];
            tc::tmem_ld16_nowait(tbase + coff + cbase + q2 * 16, raw[0]);
            if (cbase + q2 * 16 + 16 < cend) tc::tmem_ld16_nowait(tbase + coff + cbase + q2 * 16 + 16, raw[1]);
            tc::tmem_wait_ld();
#pragma unroll
        for (int qq = 0; qq < 2; qq++) {
            const int q = q2 + qq;
            const int cc = cbase + q * 16;
            if (cc >= cend) break;
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; i++) v[i] = __uint_as_float(raw[qq][i]);
            if (first && p.rs) {
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] *= rsv;
            }
            if (first && mask && live) {
                uint4 m[2];
                if (bx == H && gsm) {                 // TMA-staged gate box (SW128 layout)
                    const int gch = (cc & 63) >> 3;
                    m[0] = *reinterpret_cast<const uint4*>(gsm + tc::sw128_off(r, gch));
                    m[1] = *reinterpret_cast<const uint4*>(gsm + tc::sw128_off(r, gch + 1));
                } else {                              // gate wider than 128 columns: fetched here
                    m[0] = __ldg(msrc + (cc >> 3));
                    m[1] = __ldg(msrc + (cc >> 3) + 1);
                }
                const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(m);
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = __bfloat162float(mb[i]) > 0.f ? v[i] : 0.f;
            }
            if (first && p.relu) {
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = fmaxf(v[i], 0.f);
            }
            uint32_t o[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                o[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
            const int ch = (cc & 63) >> 3;            // 16-byte chunk within the 128-byte row
            *reinterpret_cast<uint4*>(obox + tc::sw128_off(r, ch)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(obox + tc::sw128_off(r, ch + 1)) = make_uint4(o[4], o[5], o[6], o[7]);
        }
        }
        tc::fence_proxy_async();                      // staged box -> visible to the TMA engine
        grp_bar(H);
        if (leader) {
            tma_store_2d(first ? tmC1 : tmC2, obox, cbase, tile * 128);
            bulk_commit();
        }
        ob++;
    }
}

__global__ void __launch_bounds__(kNNThreads, 1)
    k_gemm_tc_nn(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA2,
                 const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmC2,
                 const __grid_constant__ CUtensorMap tmMask, const __nv_bfloat16* __restrict__ mask, TcNN p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int kbt = p.kb1 + p.kb2;
    const int stages = p.stages;
    const uint32_t stB = p.b_stream ? (uint32_t)p.N * 128 : 0u;   // streamed weight k-block per stage
    const uint32_t st_bytes = kNNStageBytes + stB;
    uint8_t* sA = smem;
    uint8_t* sB = sA + (size_t)stages * st_bytes;                  // resident weights (not streamed)
    uint8_t* sOut = sB + (p.b_stream ? 0 : (size_t)kbt * p.N * 128);   // 2 groups x nsb boxes
    uint8_t* sMask = sOut + 2 * p.nsb * kBoxBytes;                 // [group][buf] gate boxes
    uint64_t* full = (uint64_t*)(sMask + (p.mask_tma ? 4 * kBoxBytes : 0));
    uint64_t* empty = full + kMaxNNStages;
    uint64_t* tfull = empty + kMaxNNStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* mfull = tempty + 2;                                    // [group][buf]
    uint32_t* tmem_slot = (uint32_t*)(mfull + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // weights -> shared memory once: bf16, K-major, SWIZZLE_128B, zero padded
    if (!p.b_stream) stage_weights(sB, nullptr, p.B, p.K1, p.K2, p.N, p.kb1, kbt, p.b_trans);
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < stages; s++) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; a++) { tc::mbar_init(&tfull[a], 1); tc::mbar_init(&tempty[a], 8); }
        for (int a = 0; a < 4; a++) tc::mbar_init(&mfull[a], 1);
        tc::mbar_fence_init();
        tc::tma_prefetch(&tmA1);
        if (p.kb2) tc::tma_prefetch(&tmA2);
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, p.tmem_cols);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
                for (int kb = 0; kb < kbt; kb++) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], st_bytes);
                    const bool first = kb < p.kb1;
                    uint8_t* st = sA + (size_t)stage * st_bytes;
                    tc::tma_load_2d(st, first ? &tmA1 : &tmA2, &full[stage], (first ? kb : kb - p.kb1) * 64,
                                    tile * 128);
                    if (p.b_stream) bulk_g2s(st + kNNStageBytes, p.bimg + (size_t)kb * stB, stB, &full[stage]);
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = tc::idesc_bf16(128, p.N, 0, 0);
        int stage = 0, acc = 0;
        uint32_t phase = 0, aphase = 0;
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
            tc::mbar_wait(&tempty[acc], aphase ^ 1);
            tc::fence_after();
            const uint32_t d = tmem + (uint32_t)(acc * p.N);
            for (int kb = 0; kb < kbt; kb++) {
                tc::mbar_wait(&full[stage], phase);
                tc::fence_after();
                if (lane == 0) {
                    const uint32_t a0 = tc::smem_u32(sA + (size_t)stage * st_bytes);
                    const uint32_t b0 = p.b_stream ? a0 + kNNStageBytes : tc::smem_u32(sB + (size_t)kb * p.N * 128);
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        tc::mma_f16(d, tc::smem_desc_sw128(a0 + k * 32, 0, 1024),
                                    tc::smem_desc_sw128(b0 + k * 32, 0, 1024), idesc, (kb | k) != 0);
                    tc::mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) tc::mma_commit(&tfull[acc]);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else {
        // warps 2-5 = group 0, warps 6-9 = group 1; warp & 3 = the TMEM lane quarter it may read
        const int grp = (warp - 2) >> 2;
        const int ew = warp & 3;
        const bool leader = ((warp - 2) & 3) == 0 && lane == 0;
        uint8_t* sbuf = sOut + grp * p.nsb * kBoxBytes;
        int acc = 0, ob = 0;
        uint32_t aphase = 0;
        // the row scale is fetched one tile ahead (its latency hides under a whole tile)
        auto rs_of = [&](int t) {
            const int64_t g = (int64_t)t * 128 + ew * 32 + lane;
            return (p.rs && t < p.num_tiles && g < p.M) ? __ldg(p.rs + g) : 1.f;
        };
        float rs_next = rs_of(blockIdx.x);
        // relu'-gate box of this group (C1 box grp), TMA-loaded one tile ahead, double-buffered
        const bool gated = p.mask_tma && grp < p.nb1;
        uint8_t* gbox = sMask + grp * 2 * kBoxBytes;
        uint64_t* gbar = mfull + grp * 2;
        if (gated && leader && (int)blockIdx.x < p.num_tiles) {
            tc::mbar_arrive_expect_tx(&gbar[0], kBoxBytes);
            tc::tma_load_2d(gbox, &tmMask, &gbar[0], grp * 64, blockIdx.x * 128);
        }
        int it = 0;
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, it++) {
            const uint32_t tacc = tmem + (uint32_t)(acc * p.N);
            const float rs_cur = rs_next;
            rs_next = rs_of(tile + gridDim.x);
            const uint8_t* gcur = nullptr;
            if (gated) {
                const int nb = (it + 1) & 1, next = tile + gridDim.x;
                if (leader && next < p.num_tiles) {   // its buffer was last read by tile it-1
                    tc::mbar_arrive_expect_tx(&gbar[nb], kBoxBytes);
                    tc::tma_load_2d(gbox + nb * kBoxBytes, &tmMask, &gbar[nb], grp * 64, next * 128);
                }
                tc::mbar_wait(&gbar[it & 1], (uint32_t)((it >> 1) & 1));
                gcur = gbox + (it & 1) * kBoxBytes;
            }
            if (grp == 0)
                nn_epilogue<0>(p, &tmC1, &tmC2, mask, sbuf, p.nsb, tacc, &tfull[acc], aphase, ew, lane, tile,
                               leader, ob, rs_cur, gcur);
            else
                nn_epilogue<1>(p, &tmC1, &tmC2, mask, sbuf, p.nsb, tacc, &tfull[acc], aphase, ew, lane, tile,
                               leader, ob, rs_cur, gcur);
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
        if (leader) bulk_wait_read0();
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, p.tmem_cols);
    }
}


// ------------------------------------------------------------------------- backward pair (GCN)
// One pass over a 128-row tile of dT (= Ahat dz_out) and h_in gives both backward GEMMs of a GCN
// layer: dH = (dT W^T) * relu'(h_in) [* N] (K-major operands, accumulator double-buffered in TMEM)
// and this CTA's partial of dW = h_in^T dT (MN-major operands read from the SAME shared-memory
// tiles, accumulated in TMEM over all the CTA's tiles).  The separate kernels read dT twice and
// h_in twice (once as the dW operand, once as the relu' gate); here each is read once and the
// gate comes from the staged h tile.  Partials are summed in CTA order by k_tn_reduce.
struct TcPair {
    int64_t M;
    int f_in, f_out, kbo, kbi, stages, num_tiles, nmma_w;
    const float* W;        // [f_in x f_out] fp32 (dH = dT W^T: B operand staged K-major)
    const float* rs;       // row scale of dH (N) or null
    int gate;              // relu'(h_in) gate
    float* ws;             // [grid][128][f_out] dW partials
    uint32_t tmem_cols;
};

__global__ void __launch_bounds__(kNNThreads, 1)
    k_gemm_tc_pair(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmH,
                   const __grid_constant__ CUtensorMap tmC, TcPair q) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int st_bytes = (q.kbo + q.kbi) * kBoxBytes;              // [dT boxes | h boxes]
    uint8_t* sW = smem + (size_t)q.stages * st_bytes;
    uint8_t* sOut = sW + (size_t)q.kbo * q.f_in * 128;             // 2 groups x 2 boxes
    uint64_t* full = (uint64_t*)(sOut + 4 * kBoxBytes);
    uint64_t* empty = full + kMaxNNStages;
    uint64_t* tfull = empty + kMaxNNStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* wfull = tempty + 2;
    uint32_t* tmem_slot = (uint32_t*)(wfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // W^T as the dH B operand: n = input feature (f_in rows), k = output feature, K-major
    stage_weights(sW, nullptr, q.W, q.f_out, 0, q.f_in, q.kbo, q.kbo, 1);
    if (warp == 0 && lane == 0) {
        for (int st = 0; st < q.stages; st++) { tc::mbar_init(&full[st], 1); tc::mbar_init(&empty[st], 3); }
        for (int a = 0; a < 2; a++) { tc::mbar_init(&tfull[a], 1); tc::mbar_init(&tempty[a], 8); }
        tc::mbar_init(wfull, 1);
        tc::mbar_fence_init();
        tc::tma_prefetch(&tmT);
        tc::tma_prefetch(&tmH);
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, q.tmem_cols);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tw = tmem + 2u * (uint32_t)q.f_in;              // dW accumulator columns

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < q.num_tiles; tile += gridDim.x) {
                tc::mbar_wait(&empty[stage], phase ^ 1);
                tc::mbar_arrive_expect_tx(&full[stage], st_bytes);
                uint8_t* st = smem + (size_t)stage * st_bytes;
                for (int b = 0; b < q.kbo; b++) tc::tma_load_2d(st + b * kBoxBytes, &tmT, &full[stage], b * 64, tile * 128);
                for (int b = 0; b < q.kbi; b++)
                    tc::tma_load_2d(st + (q.kbo + b) * kBoxBytes, &tmH, &full[stage], b * 64, tile * 128);
                if (++stage == q.stages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        const uint32_t id_h = tc::idesc_bf16(128, q.f_in, 0, 0);
        const uint32_t id_w = tc::idesc_bf16(128, q.nmma_w, 1, 1);
        int stage = 0, acc = 0, it = 0;
        uint32_t phase = 0, aphase = 0;
        for (int tile = blockIdx.x; tile < q.num_tiles; tile += gridDim.x, it++) {
            tc::mbar_wait(&full[stage], phase);
            tc::mbar_wait(&tempty[acc], aphase ^ 1);
            tc::fence_after();
            if (lane == 0) {
                const uint32_t sT = tc::smem_u32(smem + (size_t)stage * st_bytes);
                const uint32_t sH = sT + q.kbo * kBoxBytes;
                const uint32_t d = tmem + (uint32_t)(acc * q.f_in);
                // dH tile = dT W^T (K = output features)
                for (int kb = 0; kb < q.kbo; kb++) {
                    const uint32_t b0 = tc::smem_u32(sW + (size_t)kb * q.f_in * 128);
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        tc::mma_f16(d, tc::smem_desc_sw128(sT + kb * kBoxBytes + k * 32, 0, 1024),
                                    tc::smem_desc_sw128(b0 + k * 32, 0, 1024), id_h, (kb | k) != 0);
                }
                tc::mma_commit(&tfull[acc]);
                // dW += h^T dT over this tile's 128 rows (16 rows per MMA, MN-major operands)
#pragma unroll
                for (int k = 0; k < 8; k++)
                    tc::mma_f16(tw, tc::smem_desc_sw128(sH + k * 2048, kBoxBytes, 1024),
                                tc::smem_desc_sw128(sT + k * 2048, kBoxBytes, 1024), id_w, (it | k) != 0);
                tc::mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == q.stages) { stage = 0; phase ^= 1; }
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
        if (lane == 0) tc::mma_commit(wfull);
        __syncwarp();
    } else {
        const int grp = (warp - 2) >> 2;
        const int ew = warp & 3;
        const bool leader = ((warp - 2) & 3) == 0 && lane == 0;
        uint8_t* sbuf = sOut + grp * 2 * kBoxBytes;
        TcNN p;
        p.M = q.M; p.N = q.f_in; p.n_split = q.f_in; p.nb1 = (q.f_in + 63) / 64; p.nb2 = 0;
        p.rs = q.rs; p.relu = 0;
        int acc = 0, ob = 0, stage = 0;
        uint32_t aphase = 0, sphase = 0;
        auto rs_of = [&](int t) {
            const int64_t g = (int64_t)t * 128 + ew * 32 + lane;
            return (q.rs && t < q.num_tiles && g < q.M) ? __ldg(q.rs + g) : 1.f;
        };
        float rs_next = rs_of(blockIdx.x);
        int it = 0;
        for (int tile = blockIdx.x; tile < q.num_tiles; tile += gridDim.x, it++) {
            const uint32_t tacc = tmem + (uint32_t)(acc * q.f_in);
            const float rs_cur = rs_next;
            rs_next = rs_of(tile + gridDim.x);
            // the relu' gate: this group's h box of the tile's stage (full[stage] completed before
            // the MMA issued, and the accumulator wait below orders after that)
            const uint8_t* gcur = q.gate ? smem + (size_t)stage * st_bytes + (q.kbo + grp) * kBoxBytes : nullptr;
            if (q.gate) tc::mbar_wait(&full[stage], sphase);     // TMA-written gate visible here
            const __nv_bfloat16* gmask = q.gate ? reinterpret_cast<const __nv_bfloat16*>(gcur) : nullptr;
            if (grp == 0)
                nn_epilogue<0>(p, &tmC, &tmC, gmask, sbuf, 2, tacc, &tfull[acc], aphase, ew, lane, tile, leader,
                               ob, rs_cur, gcur);
            else
                nn_epilogue<1>(p, &tmC, &tmC, gmask, sbuf, 2, tacc, &tfull[acc], aphase, ew, lane, tile, leader,
                               ob, rs_cur, gcur);
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            grp_bar(grp);                               // the group is done with the gate box
            if (leader) tc::mbar_arrive(&empty[stage]);
            if (++stage == q.stages) { stage = 0; sphase ^= 1; }
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
        if (leader) bulk_wait_read0();
        // this CTA's dW partial: TMEM lane = input feature, columns = output features
        tc::mbar_wait(wfull, 0);
        tc::fence_after();
        const int frow = ew * 32 + lane;
        float* out = q.ws + ((int64_t)blockIdx.x * 128 + frow) * q.f_out;
        const uint32_t tb = tw + ((uint32_t)(ew * 32) << 16);
        for (int c0 = grp * 16; c0 < q.f_out; c0 += 32) {
            float v[16];
            tc::tmem_ld16(tb + c0, v);
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(out + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
        tc::fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, q.tmem_cols);
    }
}

// ------------------------------------------------------------------------------ NN, fp32 storage
// Split-fp32 transform for the fp32-storage path (1e-4 parity): every fp32 operand x is split
// into x_hi = bf16(x) and x_lo = bf16(x - x_hi) (together 16 significant bits; the residual is
// below 2^-16 |x|) and C = A_hi B_hi + A_hi B_lo + A_lo B_hi on the bf16 tensor cores (the lo*lo
// term, ~2^-18 relative, is dropped), fp32 accumulators in TMEM.  The A split cannot be done by
// TMA, so eight converter warps stream the fp32 rows with coalesced float4 loads (the next
// k-block's loads in flight while the current one is converted), write hi and lo straight into
// the K-major SWIZZLE_128B stage and arrive on the stage's mbarrier; one thread issues 3 MMAs per
// 16-wide K step; four epilogue warps apply row scale / relu'-gate / ReLU and store fp32 rows.
constexpr int kX3Conv = 8;                            // converter warps
constexpr int kX3Threads = 32 * (kX3Conv + 1 + 4);    // + MMA warp + 4 epilogue warps
constexpr int kX3StageBytes = 2 * 16384;              // hi + lo, 128 rows x 64 bf16 each
constexpr int kX3MaxStages = 4;

struct TcX3 {
    int64_t M;
    int K1, K2, N, kb1, kb2, n_split, stages, num_tiles, relu, b_trans;
    const float* A1;
    const float* A2;
    const float* B;
    const float* rs;
    const float* mask;
    float* C1;
    float* C2;
    uint32_t tmem_cols;
};

__device__ __forceinline__ void x3_split_store(uint8_t* hi_p, uint8_t* lo_p, int r, int c4, const float4& v) {
    const uint32_t hi = tc::smem_u32(hi_p), lo = tc::smem_u32(lo_p);
    const float f[4] = {v.x, v.y, v.z, v.w};
    uint32_t h[2], l[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
        const __nv_bfloat162 bh = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
        const float2 fh = __bfloat1622float2(bh);
        const __nv_bfloat162 bl = __floats2bfloat162_rn(f[2 * j] - fh.x, f[2 * j + 1] - fh.y);
        h[j] = *reinterpret_cast<const uint32_t*>(&bh);
        l[j] = *reinterpret_cast<const uint32_t*>(&bl);
    }
    const uint32_t off = tc::sw128_off(r, c4 >> 1) + (c4 & 1) * 8;
    tc::sts_v2(hi + off, h[0], h[1]);
    tc::sts_v2(lo + off, l[0], l[1]);
}

template <int IPR>
__global__ void __launch_bounds__(kX3Threads, 1)
    k_gemm_x3_nn(const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmC2, TcX3 p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int kbt = p.kb1 + p.kb2;
    uint8_t* sA = smem;
    uint8_t* sBh = sA + (size_t)p.stages * kX3StageBytes;
    uint8_t* sBl = sBh + (size_t)kbt * p.N * 128;
    uint8_t* sOut = sBl + (size_t)kbt * p.N * 128;              // 2 fp32 SW128 staging boxes
    uint64_t* full = (uint64_t*)(sOut + 2 * 16384);
    uint64_t* empty = full + kX3MaxStages;
    uint64_t* tfull = empty + kX3MaxStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    {
        stage_weights(sBh, sBl, p.B, p.K1, p.K2, p.N, p.kb1, kbt, p.b_trans);
    }
    if (threadIdx.x == 0) {
        for (int st = 0; st < p.stages; st++) { tc::mbar_init(&full[st], kX3Conv); tc::mbar_init(&empty[st], 1); }
        for (int a = 0; a < 2; a++) { tc::mbar_init(&tfull[a], 1); tc::mbar_init(&tempty[a], 4); }
        tc::mbar_fence_init();
    }
    if (warp == kX3Conv) tc::tmem_alloc(tmem_slot, p.tmem_cols);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < kX3Conv) {
        // thread t: float4 column c4 = t & 15 of the k-block, rows (t >> 4) + 16 i
        const int t = threadIdx.x, c4 = t & 15, rsub = t >> 4;
        const int items = ((p.num_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * kbt;
        auto load = [&](int it, float4 (&v)[8]) {
            const int tile = (int)blockIdx.x + (it / kbt) * (int)gridDim.x, kb = it % kbt;
            const bool first = kb < p.kb1;
            const float* A = first ? p.A1 : p.A2;
            const int Ks = first ? p.K1 : p.K2;
            const int k = (first ? kb : kb - p.kb1) * 64 + c4 * 4;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int64_t row = (int64_t)tile * 128 + rsub + 16 * i;
                v[i] = (row < p.M && k < Ks) ? __ldg(reinterpret_cast<const float4*>(A + row * Ks + k))
                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        // IPR k-blocks per round: all their loads are issued together (8 IPR float4 per thread,
        // 32 IPR KB per SM in flight), converted, and published with ONE proxy fence.  The fence
        // compiles to MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC, and the MEMBAR waits for every global
        // load still in flight -- so no load is left pending across it, and the bytes in flight
        // per round set the bandwidth (measured: 2 per round 3.3 TB/s).
        float4 v[IPR][8];
        int stage = 0;
        uint32_t phase = 0;
        for (int it = 0; it < items; it += IPR) {
            const int n = min(IPR, items - it);
#pragma unroll
            for (int j = 0; j < IPR; j++)
                if (j < n) load(it + j, v[j]);
            int st[IPR];
#pragma unroll
            for (int j = 0; j < IPR; j++) {
                if (j >= n) break;
                st[j] = stage;
                tc::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* hi = sA + (size_t)stage * kX3StageBytes;
#pragma unroll
                for (int i = 0; i < 8; i++) x3_split_store(hi, hi + 16384, rsub + 16 * i, c4, v[j][i]);
                if (++stage == p.stages) { stage = 0; phase ^= 1; }
            }
            tc::fence_proxy_async();                  // generic-proxy stores -> tensor core
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < IPR; j++)
                    if (j < n) tc::mbar_arrive(&full[st[j]]);
            }
        }
    } else if (warp == kX3Conv) {
        const uint32_t idesc = tc::idesc_bf16(128, p.N, 0, 0);
        int stage = 0, acc = 0;
        uint32_t phase = 0, aphase = 0;
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
            tc::mbar_wait(&tempty[acc], aphase ^ 1);
            tc::fence_after();
            const uint32_t d = tmem + (uint32_t)(acc * p.N);
            for (int kb = 0; kb < kbt; kb++) {
                tc::mbar_wait(&full[stage], phase);
                tc::fence_after();
                if (lane == 0) {
                    const uint32_t ah = tc::smem_u32(sA + (size_t)stage * kX3StageBytes), al = ah + 16384;
                    const uint32_t bh = tc::smem_u32(sBh + (size_t)kb * p.N * 128);
                    const uint32_t bl = tc::smem_u32(sBl + (size_t)kb * p.N * 128);
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        {
                        tc::mma_f16(d, tc::smem_desc_sw128(al + k * 32, 0, 1024),
                                    tc::smem_desc_sw128(bh + k * 32, 0, 1024), idesc, (kb | k) != 0);
                        tc::mma_f16(d, tc::smem_desc_sw128(ah + k * 32, 0, 1024),
                                    tc::smem_desc_sw128(bl + k * 32, 0, 1024), idesc, 1);
                        }
                        tc::mma_f16(d, tc::smem_desc_sw128(ah + k * 32, 0, 1024),
                                    tc::smem_desc_sw128(bh + k * 32, 0, 1024), idesc, 1);
                    }
                    tc::mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == p.stages) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) tc::mma_commit(&tfull[acc]);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else {
        // epilogue: per 32-column output box, TMEM -> registers -> row scale / relu'-gate /
        // ReLU -> SW128 fp32 staging box (double-buffered) -> TMA bulk-tensor store (coalesced;
        // rows past M and columns past the tensor edge are clipped by the TMA unit)
        const int ew = warp & 3;
        const int r = ew * 32 + lane;
        const uint32_t tq = (uint32_t)(ew * 32) << 16;
        const bool leader = warp == kX3Conv + 1 && lane == 0;
        const int nb1 = (p.n_split + 31) >> 5, nb2 = (p.N - p.n_split + 31) >> 5;
        int acc = 0, ob = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
            const int64_t grow = (int64_t)tile * 128 + r;
            const bool live = grow < p.M;
            const float rsv = (p.rs && live) ? __ldg(p.rs + grow) : 1.f;
            tc::mbar_wait(&tfull[acc], aphase);
            tc::fence_after();
            const uint32_t tb = tmem + (uint32_t)(acc * p.N) + tq;
            for (int bx = 0; bx < nb1 + nb2; bx++) {
                const bool first = bx < nb1;
                const int cbase = first ? bx * 32 : (bx - nb1) * 32;          // column in C1 / C2
                const int cend = first ? min(cbase + 32, p.n_split) : min(cbase + 32, p.N - p.n_split);
                const int coff = first ? 0 : p.n_split;                        // accumulator column
                uint8_t* obox = sOut + (ob & 1) * 16384;
                if (leader) bulk_wait_read1();        // the store that last used this buffer is done
                epi_bar();
                for (int h = 0; h < 2; h++) {
                    const int cc = cbase + h * 16;
                    if (cc >= cend) break;
                    float v[16];
                    tc::tmem_ld16(tb + coff + cc, v);
                    if (first) {
                        if (p.rs) {
#pragma unroll
                            for (int i = 0; i < 16; i++) v[i] *= rsv;
                        }
                        if (p.mask && live) {
                            const float4* mk = reinterpret_cast<const float4*>(p.mask + grow * p.n_split + cc);
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                const float4 m = __ldg(mk + q);
                                v[4 * q] = m.x > 0.f ? v[4 * q] : 0.f;
                                v[4 * q + 1] = m.y > 0.f ? v[4 * q + 1] : 0.f;
                                v[4 * q + 2] = m.z > 0.f ? v[4 * q + 2] : 0.f;
                                v[4 * q + 3] = m.w > 0.f ? v[4 * q + 3] : 0.f;
                            }
                        }
                        if (p.relu) {
#pragma unroll
                            for (int i = 0; i < 16; i++) v[i] = fmaxf(v[i], 0.f);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        tc::sts_v4(tc::smem_u32(obox) + tc::sw128_off(r, h * 4 + q), v[4 * q], v[4 * q + 1],
                                   v[4 * q + 2], v[4 * q + 3]);
                }
                tc::fence_proxy_async();              // staged box -> visible to the TMA engine
                epi_bar();
                if (leader) {
                    tma_store_2d(first ? &tmC1 : &tmC2, obox, cbase, tile * 128);
                    bulk_commit();
                }
                ob++;
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
        if (leader) bulk_wait_read0();
    }
    __syncthreads();
    if (warp == kX3Conv) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, p.tmem_cols);
    }
}


// Split-fp32 weight gradient (fp32 storage): dW partial of one (row slab, 128-feature tile) =
// A_hi^T B_hi + A_hi^T B_lo + A_lo^T B_hi over the slab, both operands MN-major (node rows are
// the reduction dimension), split by the converter warps into the SW128 boxes TMA would write
// for bf16 (64 node rows x 64 columns per box).  Same slab plan, workspace and fixed-order
// reduction (k_tn_reduce) as the bf16 kernel.
struct TcX3TN {
    int64_t M;
    int K1, K2, N, Nmma, ft1, nbox_b, slabs, stages;
    int64_t rows_per_slab;
    const float* A1;
    const float* A2;
    const float* B;
    float* ws;
    uint32_t tmem_cols;
};

__global__ void __launch_bounds__(kX3Threads, 1) k_gemm_x3_tn(TcX3TN p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int a_bytes = 2 * 8192, b_bytes = p.nbox_b * 8192;
    const int st_bytes = 2 * (a_bytes + b_bytes);        // [A hi | A lo | B hi | B lo]
    uint64_t* full = (uint64_t*)(smem + (size_t)p.stages * st_bytes);
    uint64_t* empty = full + kX3MaxStages;
    uint64_t* tfull = empty + kX3MaxStages;
    uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ft = blockIdx.y;
    const bool src1 = ft < p.ft1;
    const float* A = src1 ? p.A1 : p.A2;
    const int Ks = src1 ? p.K1 : p.K2;
    const int fbase = (src1 ? ft : ft - p.ft1) * 128;
    const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_slab;
    const int64_t r1 = min(p.M, r0 + p.rows_per_slab);
    const int nkb = r1 > r0 ? (int)ceil_div(r1 - r0, 64) : 0;

    if (threadIdx.x == 0) {
        for (int st = 0; st < p.stages; st++) { tc::mbar_init(&full[st], kX3Conv); tc::mbar_init(&empty[st], 1); }
        tc::mbar_init(tfull, 1);
        tc::mbar_fence_init();
    }
    if (warp == kX3Conv) tc::tmem_alloc(tmem_slot, p.tmem_cols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < kX3Conv) {
        const int t = threadIdx.x, c4 = t & 15, rr = t >> 4;     // rows rr + 16 i, i < 4
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < nkb; kb++) {
            const int64_t rowb = r0 + (int64_t)kb * 64;
            float4 va[2][4], vb[4][4];
#pragma unroll
            for (int bx = 0; bx < 2; bx++) {
                const int f = fbase + bx * 64 + c4 * 4;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int64_t row = rowb + rr + 16 * i;
                    va[bx][i] = (row < r1 && f < Ks) ? __ldg(reinterpret_cast<const float4*>(A + row * Ks + f))
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int bx = 0; bx < 4; bx++) {
                const int n = bx * 64 + c4 * 4;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int64_t row = rowb + rr + 16 * i;
                    vb[bx][i] = (bx < p.nbox_b && row < r1 && n < p.N)
                                    ? __ldg(reinterpret_cast<const float4*>(p.B + row * p.N + n))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            tc::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + (size_t)stage * st_bytes;
#pragma unroll
            for (int bx = 0; bx < 2; bx++)
#pragma unroll
                for (int i = 0; i < 4; i++)
                    x3_split_store(st + bx * 8192, st + a_bytes + bx * 8192, rr + 16 * i, c4, va[bx][i]);
#pragma unroll
            for (int bx = 0; bx < 4; bx++) {
                if (bx >= p.nbox_b) break;
#pragma unroll
                for (int i = 0; i < 4; i++)
                    x3_split_store(st + 2 * a_bytes + bx * 8192, st + 2 * a_bytes + b_bytes + bx * 8192, rr + 16 * i,
                                   c4, vb[bx][i]);
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[stage]);
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
    } else if (warp == kX3Conv) {
        const uint32_t idesc = tc::idesc_bf16(128, p.Nmma, 1, 1);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < nkb; kb++) {
            tc::mbar_wait(&full[stage], phase);
            tc::fence_after();
            if (lane == 0) {
                const uint32_t ah = tc::smem_u32(smem + (size_t)stage * st_bytes), al = ah + a_bytes;
                const uint32_t bh = ah + 2 * a_bytes, bl = bh + b_bytes;
#pragma unroll
                for (int k = 0; k < 4; k++) {      // 16 node rows per MMA = two 8-row K groups
                    tc::mma_f16(tmem, tc::smem_desc_sw128(al + k * 2048, 8192, 1024),
                                tc::smem_desc_sw128(bh + k * 2048, 8192, 1024), idesc, (kb | k) != 0);
                    tc::mma_f16(tmem, tc::smem_desc_sw128(ah + k * 2048, 8192, 1024),
                                tc::smem_desc_sw128(bl + k * 2048, 8192, 1024), idesc, 1);
                    tc::mma_f16(tmem, tc::smem_desc_sw128(ah + k * 2048, 8192, 1024),
                                tc::smem_desc_sw128(bh + k * 2048, 8192, 1024), idesc, 1);
                }
                tc::mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) tc::mma_commit(tfull);
        __syncwarp();
    } else {
        const int ew = warp & 3;
        const int frow = ew * 32 + lane;
        if (nkb > 0) {
            tc::mbar_wait(tfull, 0);
            tc::fence_after();
        }
        float* out = p.ws + (((int64_t)blockIdx.x * gridDim.y + ft) * 128 + frow) * p.N;
        const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16);
        for (int c0 = 0; c0 < p.N; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tbase + c0, v);
            if (nkb == 0) {
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(out + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
        tc::fence_before();
    }
    __syncthreads();
    if (warp == kX3Conv) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, p.tmem_cols);
    }
}

// ------------------------------------------------------------------------------------- TN
struct TcTN {
    int64_t M;
    int K1, K2, N, Nmma, ft1, ft2, nbox_b;
    int64_t rows_per_slab;
    int slabs;
    int stages;         // ring depth (fills shared memory, <= kTNMaxStages)
    float* ws;          // [slabs][ftiles][128][N]
    uint32_t tmem_cols;
};

__global__ void __launch_bounds__(kTcThreads, 1)
    k_gemm_tc_tn(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA2,
                 const __grid_constant__ CUtensorMap tmB, TcTN p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int a_bytes = 2 * 8192, b_bytes = p.nbox_b * 8192, st_bytes = a_bytes + b_bytes;
    const int kTNStages = p.stages;
    uint64_t* full = (uint64_t*)(smem + (size_t)kTNStages * st_bytes);
    uint64_t* empty = full + kTNMaxStages;
    uint64_t* tfull = empty + kTNStages;
    uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ft = blockIdx.y;
    const bool src1 = ft < p.ft1;
    const int fbase = (src1 ? ft : ft - p.ft1) * 128;
    const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_slab;
    const int64_t r1 = min(p.M, r0 + p.rows_per_slab);
    const int nkb = r1 > r0 ? (int)ceil_div(r1 - r0, 64) : 0;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kTNStages; s++) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_init(tfull, 1);
        tc::mbar_fence_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, p.tmem_cols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const CUtensorMap* ma = src1 ? &tmA1 : &tmA2;
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = 0; kb < nkb; kb++) {
                tc::mbar_wait(&empty[stage], phase ^ 1);
                tc::mbar_arrive_expect_tx(&full[stage], st_bytes);
                uint8_t* st = smem + (size_t)stage * st_bytes;
                const int y = (int)(r0 + kb * 64);
                tc::tma_load_2d(st, ma, &full[stage], fbase, y);
                tc::tma_load_2d(st + 8192, ma, &full[stage], fbase + 64, y);
                for (int j = 0; j < p.nbox_b; j++)
                    tc::tma_load_2d(st + a_bytes + j * 8192, &tmB, &full[stage], j * 64, y);
                if (++stage == kTNStages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = tc::idesc_bf16(128, p.Nmma, 1, 1);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < nkb; kb++) {
            tc::mbar_wait(&full[stage], phase);
            tc::fence_after();
            if (lane == 0) {
                const uint32_t a0 = tc::smem_u32(smem + (size_t)stage * st_bytes);
                const uint32_t b0 = a0 + a_bytes;
#pragma unroll
                for (int k = 0; k < 4; k++)      // 16 node rows per MMA = two 8-row K groups
                    tc::mma_f16(tmem, tc::smem_desc_sw128(a0 + k * 2048, 8192, 1024),
                                tc::smem_desc_sw128(b0 + k * 2048, 8192, 1024), idesc, (kb | k) != 0);
                tc::mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == kTNStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) tc::mma_commit(tfull);
        __syncwarp();
    } else {
        const int ew = warp & 3;
        const int frow = ew * 32 + lane;
        if (nkb > 0) {
            tc::mbar_wait(tfull, 0);
            tc::fence_after();
        }
        float* out = p.ws + (((int64_t)blockIdx.x * gridDim.y + ft) * 128 + frow) * p.N;
        const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16);
        for (int c0 = 0; c0 < p.N; c0 += 16) {
            float v[16];
            tc::tmem_ld16(tbase + c0, v);
            if (nkb == 0) {
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(out + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
        tc::fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, p.tmem_cols);
    }
}

// dW[r][n] = sum_slab ws[slab][ft(r)][row(r)][n].  Block = 32 outputs x kRedGroups slab groups:
// thread (o, g) sums slabs g, g + kRedGroups, ... in order (a few independent loads in flight),
// then the group sums are added in group order -- a fixed summation tree, so the result is
// bitwise deterministic.
// A/B knobs (grappa_set_kernel_variant "tnstages" / "tnred"): ring depth (0 = fill shared
// memory) and slab groups of the reduction (8 or 32)
// ring depth of the weight-gradient GEMM: 4 stages measured best (6-7 and a full-smem ring were
// slower), and an 8-group fixed-order split-K reduction (32 groups measured no faster)
constexpr int kTnStages = 4;
template <int kRedGroups>
__global__ void __launch_bounds__(32 * kRedGroups) k_tn_reduce(int64_t count, int N, int K1, int K2, int ft1,
                                                               int ftiles, int slabs, const float* __restrict__ ws,
                                                               float* __restrict__ dw) {
    __shared__ float part[kRedGroups][33];
    const int o = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + o;
    float s = 0.f;
    if (i < count) {
        const int r = (int)(i / N), n = (int)(i % N);
        int ft, row;
        if (r < K1) { ft = r / 128; row = r % 128; }
        else { ft = ft1 + (r - K1) / 128; row = (r - K1) % 128; }
        const float* src = ws + ((int64_t)ft * 128 + row) * N + n;
        const int64_t zstride = (int64_t)ftiles * 128 * N;
#pragma unroll 4
        for (int z = g; z < slabs; z += kRedGroups) s += src[(int64_t)z * zstride];
    }
    part[g][o] = s;
    __syncthreads();
    if (g == 0 && i < count) {
        float t = 0.f;
        for (int k = 0; k < kRedGroups; k++) t += part[k][o];
        dw[i] = t;
    }
}

// ------------------------------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static grappa_status get_encoder() {
    if (g_encode) return GRAPPA_OK;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return GRAPPA_E_CUDA;
    }
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    return GRAPPA_OK;
}

// 2-D bf16 row-major [rows x cols] map, box {64 cols, box_rows rows}, SWIZZLE_128B
static grappa_status make_map(CUtensorMap* m, const void* ptr, int64_t rows, int cols, int box_rows,
                              bool f32 = false) {
    GRAPPA_TRY(get_encoder());
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)cols * (f32 ? 4 : 2)};
    cuuint32_t box[2] = {f32 ? 32u : 64u, (cuuint32_t)box_rows};     // 128-byte box rows
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                          const_cast<void*>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%d", (int)r, (long long)rows, cols);
        return GRAPPA_E_CUDA;
    }
    return GRAPPA_OK;
}

// row-gather map of a bf16 row-major [rows x cols] tensor for tile::gather4: box {cols, 1} (each
// gather4 writes 4 whole rows contiguously), no swizzle (spmm_tma.cu)
grappa_status tma_map_rows_bf16(CUtensorMap* m, const void* ptr, int64_t rows, int cols) {
    GRAPPA_TRY(get_encoder());
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)cols, 1u};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (row gather) failed (%d): rows=%lld cols=%d", (int)r, (long long)rows, cols);
        return GRAPPA_E_CUDA;
    }
    return GRAPPA_OK;
}

// A ring + resident weights + 2 groups x nsb staging boxes + barriers; the deepest ring
// (<= 8 stages) and double-buffered staging when they fit
static size_t nn_smem_of(int kbt, int N, int stages, int nsb, int mask_tma, int b_stream = 0) {
    const size_t stage = kNNStageBytes + (b_stream ? (size_t)N * 128 : 0);
    return 1024 + (size_t)stages * stage + (b_stream ? 0 : (size_t)kbt * N * 128) + (size_t)2 * nsb * kBoxBytes +
           (mask_tma ? (size_t)4 * kBoxBytes : 0) + 256;
}
// resident weights when they fit next to a ring of >= 2 stages, else streamed weight k-blocks
static bool nn_plan(int kbt, int N, int mask_tma, int* stages, int* nsb, int* b_stream, int prefer_stream = 0) {
    for (int bs = prefer_stream; bs <= 1; bs++)
        for (int b = 2; b >= 1; b--)
            for (int st = kMaxNNStages; st >= 2; st--)
                if (nn_smem_of(kbt, N, st, b, mask_tma, bs) <= (size_t)kMaxSmem && (b == 1 || st >= 4)) {
                    *stages = st;
                    *nsb = b;
                    *b_stream = bs;
                    return true;
                }
    return false;
}

bool gemm_tc_nn_supported(const GemmArgs& g) {
    const int kbt = (int)(ceil_div(g.K1, 64) + ceil_div(g.K2, 64));
    int st, nsb, bs;
    return g.N % 16 == 0 && g.N <= 256 && g.n_split % 16 == 0 && g.K1 % 8 == 0 && g.K2 % 8 == 0 &&
           nn_plan(kbt, g.N, 0, &st, &nsb, &bs) && g.M < (1ll << 31);
}

static uint32_t pow2_cols(int c) {
    uint32_t n = 32;
    while ((int)n < c) n <<= 1;
    return n;
}

grappa_status gemm_tc_nn(grappa_ctx* ctx, const GemmArgs& g, cudaStream_t s) {
    CUtensorMap m1, m2, c1, c2;
    GRAPPA_TRY(make_map(&m1, g.A1, g.M, g.K1, 128));
    if (g.K2 > 0) GRAPPA_TRY(make_map(&m2, g.A2, g.M, g.K2, 128));
    else m2 = m1;
    GRAPPA_TRY(make_map(&c1, g.C1, g.M, g.n_split, 128));
    if (g.N > g.n_split) GRAPPA_TRY(make_map(&c2, g.C2, g.M, g.N - g.n_split, 128));
    else c2 = c1;
    TcNN p;
    p.M = g.M; p.K1 = g.K1; p.K2 = g.K2; p.N = g.N;
    p.kb1 = (int)ceil_div(g.K1, 64); p.kb2 = (int)ceil_div(g.K2, 64);
    p.B = g.B; p.rs = g.row_scale; p.b_trans = g.b_trans; p.relu = g.relu;
    p.has_mask = g.mask != nullptr; p.n_split = g.n_split;
    p.nb1 = (int)ceil_div(g.n_split, 64); p.nb2 = (int)ceil_div(g.N - g.n_split, 64);
    p.num_tiles = (int)ceil_div(g.M, 128);
    p.tmem_cols = pow2_cols(2 * g.N);
    // few tiles per CTA (mini-batch blocks): the per-CTA fp32 -> bf16 staging of the whole weight
    // is not amortised (ncu: ~half of a 19 us call at M = 10^4), so the weight is converted once
    // into the SW128 image (k_weight_image) and streamed per k-block by bulk copies instead
    const int prefer_stream = (ctx->var_gemm_stream == 1 || (ctx->var_gemm_stream == 0 &&
                               p.num_tiles <= 2 * (int64_t)ctx->sm_count)) ? 1 : 0;
    // relu'-gate through TMA when each epilogue group owns at most one gated box and it fits
    p.mask_tma = p.has_mask && p.nb1 <= 2 &&
                 nn_plan(p.kb1 + p.kb2, g.N, 1, &p.stages, &p.nsb, &p.b_stream, prefer_stream) ? 1 : 0;
    if (!p.mask_tma && !nn_plan(p.kb1 + p.kb2, g.N, 0, &p.stages, &p.nsb, &p.b_stream, prefer_stream)) {
        set_error("gemm_tc_nn: shape does not fit shared memory");
        return GRAPPA_E_SUPPORT;
    }
    p.bimg = nullptr;
    if (p.b_stream) {            // the weight image, once per call (stream-ordered before the GEMM)
        const int kbt = p.kb1 + p.kb2;
        GRAPPA_TRY(ctx->wimg.grow((size_t)kbt * g.N * 128));
        k_weight_image<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)kbt * 8 * g.N, 256), (int64_t)ctx->sm_count * 4),
                         256, 0, s>>>(g.B, g.K1, g.K2, g.N, p.kb1, kbt, g.b_trans, (uint8_t*)ctx->wimg.p);
        GRAPPA_LAUNCHED(ctx);
        p.bimg = (const uint8_t*)ctx->wimg.p;
    }
    CUtensorMap mk;
    if (p.mask_tma) GRAPPA_TRY(make_map(&mk, g.mask, g.M, g.n_split, 128));
    else mk = c1;
    const size_t smem = nn_smem_of(p.kb1 + p.kb2, g.N, p.stages, p.nsb, p.mask_tma, p.b_stream);
    static bool attr = false;
    if (!attr) {
        GRAPPA_CUDA(cudaFuncSetAttribute(k_gemm_tc_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        attr = true;
    }
    const int grid = (int)std::min<int64_t>(p.num_tiles, ctx->sm_count);
    k_gemm_tc_nn<<<grid, kNNThreads, smem, s>>>(m1, m2, c1, c2, mk, (const __nv_bfloat16*)g.mask, p);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}


// split-fp32 NN (fp32 storage): resident hi + lo weights, 2..4 A stages
static size_t x3_smem_of(int kbt, int N, int stages) {
    return 1024 + (size_t)stages * kX3StageBytes + (size_t)2 * kbt * N * 128 + 2 * 16384 + 256;
}
static int x3_stages(int kbt, int N) {
    for (int st = kX3MaxStages; st >= 2; st--)
        if (x3_smem_of(kbt, N, st) <= (size_t)kMaxSmem) return st;
    return 0;
}
bool gemm_x3_nn_supported(const GemmArgs& g) {
    const int kbt = (int)(ceil_div(g.K1, 64) + ceil_div(g.K2, 64));
    return g.N % 16 == 0 && g.N <= 256 && g.n_split % 16 == 0 && g.K1 % 4 == 0 && g.K2 % 4 == 0 &&
           x3_stages(kbt, g.N) >= 2 && g.M < (1ll << 31);
}
grappa_status gemm_x3_nn(grappa_ctx* ctx, const GemmArgs& g, cudaStream_t s) {
    TcX3 p;
    p.M = g.M; p.K1 = g.K1; p.K2 = g.K2; p.N = g.N;
    p.kb1 = (int)ceil_div(g.K1, 64); p.kb2 = (int)ceil_div(g.K2, 64);
    p.n_split = g.n_split; p.relu = g.relu; p.b_trans = g.b_trans;
    p.stages = x3_stages(p.kb1 + p.kb2, g.N);
    p.num_tiles = (int)ceil_div(g.M, 128);
    p.A1 = (const float*)g.A1; p.A2 = (const float*)g.A2; p.B = g.B; p.rs = g.row_scale;
    p.mask = (const float*)g.mask; p.C1 = (float*)g.C1; p.C2 = (float*)g.C2;
    p.tmem_cols = pow2_cols(2 * g.N);
    static bool attr = false;
    if (!attr) {
        GRAPPA_CUDA(cudaFuncSetAttribute(k_gemm_x3_nn<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        GRAPPA_CUDA(cudaFuncSetAttribute(k_gemm_x3_nn<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        attr = true;
    }
    CUtensorMap c1, c2;
    GRAPPA_TRY(make_map(&c1, g.C1, g.M, g.n_split, 128, true));
    if (g.N > g.n_split) GRAPPA_TRY(make_map(&c2, g.C2, g.M, g.N - g.n_split, 128, true));
    else c2 = c1;
    const int grid = (int)std::min<int64_t>(p.num_tiles, ctx->sm_count);
    const size_t smem = x3_smem_of(p.kb1 + p.kb2, g.N, p.stages);
    if (p.stages >= 3) k_gemm_x3_nn<3><<<grid, kX3Threads, smem, s>>>(c1, c2, p);
    else k_gemm_x3_nn<2><<<grid, kX3Threads, smem, s>>>(c1, c2, p);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}


static int tn_ftiles(int K) { return (int)ceil_div(K, 128); }

static void tn_plan(int64_t M, int ftiles, int sm_count, int* slabs, int64_t* rps) {
    int s = sm_count / ftiles;
    if (s < 1) s = 1;
    int64_t r = ceil_div(ceil_div(M > 0 ? M : 1, s), 64) * 64;
    *rps = r;
    *slabs = (int)ceil_div(M > 0 ? M : 1, r);
}

// backward pair (GCN, bf16): dz_in = (dT W^T) * relu'(h_in) [* rs] and dW = h_in^T dT
static size_t pair_smem_of(int kbo, int kbi, int f_in, int stages) {
    return 1024 + (size_t)stages * (kbo + kbi) * kBoxBytes + (size_t)kbo * f_in * 128 + 4 * kBoxBytes + 256;
}
bool gemm_tc_pair_supported(int64_t M, int f_in, int f_out) {
    if (f_in <= 64 || f_in > 128 || f_in % 16 || f_out > 128 || f_out % 16 || M >= (1ll << 31)) return false;
    const int kbo = (f_out + 63) / 64;
    return pair_smem_of(kbo, 2, f_in, 2) <= (size_t)kMaxSmem;
}
grappa_status gemm_tc_pair(grappa_ctx* ctx, int64_t M, int f_in, int f_out, const void* dT, const void* h,
                           const float* W, const float* rs, int gate, void* dz_in, float* ws, float* dw,
                           cudaStream_t s) {
    CUtensorMap mt, mh, mc;
    GRAPPA_TRY(make_map(&mt, dT, M, f_out, 128));
    GRAPPA_TRY(make_map(&mh, h, M, f_in, 128));
    GRAPPA_TRY(make_map(&mc, dz_in, M, f_in, 128));
    TcPair q;
    q.M = M; q.f_in = f_in; q.f_out = f_out;
    q.kbo = (f_out + 63) / 64; q.kbi = 2;
    q.nmma_w = q.kbo * 64;
    q.W = W; q.rs = rs; q.gate = gate; q.ws = ws;
    q.num_tiles = (int)ceil_div(M, 128);
    q.tmem_cols = 512;
    q.stages = 2;
    while (q.stages < 4 && pair_smem_of(q.kbo, q.kbi, f_in, q.stages + 1) <= (size_t)kMaxSmem) q.stages++;
    // the dW split: CTA b owns tiles b, b + grid, ... (grid fixed by M: deterministic sums)
    int slabs;
    int64_t rps;
    tn_plan(M, 1, kTnCtas, &slabs, &rps);
    const int grid = (int)std::min<int64_t>(q.num_tiles, slabs);
    static bool attr = false;
    if (!attr) {
        GRAPPA_CUDA(cudaFuncSetAttribute(k_gemm_tc_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        attr = true;
    }
    k_gemm_tc_pair<<<grid, kNNThreads, pair_smem_of(q.kbo, q.kbi, f_in, q.stages), s>>>(mt, mh, mc, q);
    GRAPPA_LAUNCHED(ctx);
    const int64_t count = (int64_t)f_in * f_out;
    k_tn_reduce<8><<<(unsigned)ceil_div(count, 32), 32 * 8, 0, s>>>(count, f_out, f_in, 0, 1, 1, grid, ws, dw);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}


size_t gemm_tc_tn_ws_bytes(int64_t M, int K1, int K2, int N) {
    const int ft = tn_ftiles(K1) + (K2 ? tn_ftiles(K2) : 0);
    int slabs;
    int64_t rps;
    tn_plan(M, ft, kTnCtas, &slabs, &rps);
    return (size_t)slabs * ft * 128 * N * sizeof(float);
}

bool gemm_tc_tn_supported(const GemmTNArgs& g) {
    return g.N % 16 == 0 && g.N <= 256 && g.K1 % 8 == 0 && g.K2 % 8 == 0 && g.M < (1ll << 31);
}

grappa_status gemm_tc_tn(grappa_ctx* ctx, const GemmTNArgs& g, cudaStream_t s) {
    CUtensorMap m1, m2, mb;
    GRAPPA_TRY(make_map(&m1, g.A1, g.M, g.K1, 64));
    if (g.K2 > 0) GRAPPA_TRY(make_map(&m2, g.A2, g.M, g.K2, 64));
    else m2 = m1;
    GRAPPA_TRY(make_map(&mb, g.B, g.M, g.N, 64));
    TcTN p;
    p.M = g.M; p.K1 = g.K1; p.K2 = g.K2; p.N = g.N;
    p.Nmma = (int)ceil_div(g.N, 64) * 64;
    p.nbox_b = p.Nmma / 64;
    p.ft1 = tn_ftiles(g.K1);
    p.ft2 = g.K2 ? tn_ftiles(g.K2) : 0;
    const int ftiles = p.ft1 + p.ft2;
    tn_plan(g.M, ftiles, kTnCtas, &p.slabs, &p.rows_per_slab);
    p.ws = g.ws;
    p.tmem_cols = pow2_cols(p.Nmma);
    const size_t st_bytes = 16384 + (size_t)p.nbox_b * 8192;
    p.stages = (int)std::min<size_t>(kTNMaxStages, (kMaxSmem - 1024 - 512) / st_bytes);
    p.stages = std::min(p.stages, kTnStages);
    const size_t smem = 1024 + (size_t)p.stages * st_bytes + 512;
    static bool attr = false;
    if (!attr) {
        GRAPPA_CUDA(cudaFuncSetAttribute(k_gemm_tc_tn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        attr = true;
    }
    dim3 grid(p.slabs, ftiles);
    k_gemm_tc_tn<<<grid, kTcThreads, smem, s>>>(m1, m2, mb, p);
    GRAPPA_LAUNCHED(ctx);
    const int64_t count = (int64_t)(g.K1 + g.K2) * g.N;
    k_tn_reduce<8><<<(unsigned)ceil_div(count, 32), 32 * 8, 0, s>>>(count, g.N, g.K1, g.K2, p.ft1, ftiles,
                                                                   p.slabs, g.ws, g.C);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}


bool gemm_x3_tn_supported(const GemmTNArgs& g) {
    return g.N % 16 == 0 && g.N <= 256 && g.K1 % 4 == 0 && g.K2 % 4 == 0 && g.M < (1ll << 31);
}
grappa_status gemm_x3_tn(grappa_ctx* ctx, const GemmTNArgs& g, cudaStream_t s) {
    TcX3TN p;
    p.M = g.M; p.K1 = g.K1; p.K2 = g.K2; p.N = g.N;
    p.Nmma = (int)ceil_div(g.N, 64) * 64;
    p.nbox_b = p.Nmma / 64;
    p.ft1 = tn_ftiles(g.K1);
    const int ftiles = p.ft1 + (g.K2 ? tn_ftiles(g.K2) : 0);
    tn_plan(g.M, ftiles, kTnCtas, &p.slabs, &p.rows_per_slab);
    p.A1 = (const float*)g.A1; p.A2 = (const float*)g.A2; p.B = (const float*)g.B; p.ws = g.ws;
    p.tmem_cols = pow2_cols(p.Nmma);
    const size_t st_bytes = 2 * (16384 + (size_t)p.nbox_b * 8192);
    p.stages = (int)std::min<size_t>(kX3MaxStages, (kMaxSmem - 1024 - 512) / st_bytes);
    const size_t smem = 1024 + (size_t)p.stages * st_bytes + 512;
    static bool attr = false;
    if (!attr) {
        GRAPPA_CUDA(cudaFuncSetAttribute(k_gemm_x3_tn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        attr = true;
    }
    dim3 grid(p.slabs, ftiles);
    k_gemm_x3_tn<<<grid, kX3Threads, smem, s>>>(p);
    GRAPPA_LAUNCHED(ctx);
    const int64_t count = (int64_t)(g.K1 + g.K2) * g.N;
    k_tn_reduce<8><<<(unsigned)ceil_div(count, 32), 32 * 8, 0, s>>>(count, g.N, g.K1, g.K2, p.ft1, ftiles, p.slabs,
                                                                   g.ws, g.C);
    GRAPPA_LAUNCHED(ctx);
    return GRAPPA_OK;
}

}  // namespace grappa
