// consensus_tma.cuh -- persistent, TMA-pipelined consensus pass (K2) for
// uniform tilings with 64- or 128-wide blocks.  Included by dope_lattice.cu
// inside namespace dope (uses Lat2, CtaAgg, pass_tail, other_buffer).
//
// Same arithmetic as k_consensus_vec (solve_global + clamp admm.py:136-180,
// update_multipliers admm.py:183-190, block residuals admm.py:193-199, energy
// of the previous iterate energy.py:187-194), organised for HBM:
//   * persistent grid (a few CTAs per SM); each CTA walks its blocks as tiles
//     of TH x TW pixels (64x64, or 32 rows of a 128-wide block);
//   * per tile, one thread issues 2D TMA loads (cp.async.bulk.tensor) of the
//     int16 multipliers, the uint8 iterate y2 (+ the row below), the y2
//     column right of the tile and the label tile with a 1-row / 16-byte halo
//     into a STAGES-deep shared-memory ring, completion tracked by mbarriers;
//     u is not streamed (the unary energy is kept incrementally);
//   * results go straight from registers to HBM (8-byte multiplier quads,
//     4-byte iterate quads);
//   * per-block partials are accumulated with one atomic per warp (the next
//     K1 clears them); each CTA then folds its own blocks into pass-wide
//     aggregates, so the last CTA only adds up one residual sum per CTA.

struct TmaMaps {
    CUtensorMap a, y[3], yr[3], yhat;
    CUtensorMap yrow[3];      // y2: one row of TW (ring-only tiles)
    CUtensorMap h16;          // labels: 16 bytes of one row (ring-only corners)
    CUtensorMap hrow, hcol;   // labels: one row of TW, a 16-byte column of TH rows
    CUtensorMap arow, acol;   // multipliers: one row of TW, an 8-wide column of TH rows
};

// Stage layout of one TH x TW tile.
// Solved block (re-solved by this iteration's K1): multipliers (int16),
// previous iterate y2 (uint8, +1 row below), the 16-byte column right of the
// tile (its first byte is the right-halo y2), labels with a 1-row / 16-byte
// halo.
// Clean block (not re-solved): its interior is a fixed point of the update
// (y == yhat there and neither moves), so only y2 and the
// labels just across the block boundary are streamed (its own labels equal
// y2 / 2); ring multipliers are read directly.
// u is never streamed: the unary energy is kept incrementally.
template <int TW, int TH_, int NT_ = 128, int STAGES_ = 8>
struct TmaCfg {
    static constexpr int TH = TH_;                       // tile rows
    static constexpr int NT = NT_;
    static constexpr int QPT = TH * TW / 4 / NT;         // quads per thread
    static_assert(QPT >= 1 && QPT * NT * 4 == TH * TW, "whole quads per thread");
    static_assert(TH % 8 == 0, "128-byte aligned clean boxes");
    static constexpr int YHW = TW + 32;                  // label box width (bytes)
    static constexpr int B_A = TW * TH * 2;
    static constexpr int B_Y = TW * (TH + 1);
    static constexpr int B_YR = 16 * TH;
    static constexpr int B_H = YHW * (TH + 2);
    static constexpr int O_A = 0;
    static constexpr int O_Y = (O_A + B_A + 127) / 128 * 128;
    static constexpr int O_YR = (O_Y + B_Y + 127) / 128 * 128;
    static constexpr int O_H = (O_YR + B_YR + 127) / 128 * 128;
    static constexpr int STAGE = (O_H + B_H + 127) / 128 * 128;
    static constexpr int TX = B_A + B_Y + B_YR + B_H;
    // clean tiles: neighbour labels and the ring multipliers (8-wide
    // columns at both edges, first / last row) in the unused multiplier area
    static constexpr int O_HUP = O_A, O_HDN = O_A + 128, O_HL = O_A + 256, O_HR = O_HL + 16 * TH;
    static constexpr int O_AL = O_HR + 16 * TH, O_AR = O_AL + 16 * TH;
    static constexpr int O_AT = O_AR + 16 * TH, O_AB = O_AT + 2 * TW;
    static_assert(O_AB + 2 * TW <= O_Y, "clean boxes fit the multiplier area");
    static constexpr int TX_CLEAN = B_Y + B_YR + 2 * TW + 2 * 16 * TH + 2 * 16 * TH + 2 * 2 * TW;
    // ring-only tiles (clean block whose energy partial and output-buffer
    // copy both still hold): the ring's own y2 (16-byte
    // columns, rows) and the corner labels, in the (unused) y2 / label area
    static constexpr int RW = (TW + 127) / 128 * 128;
    static constexpr int O_YCL = O_Y, O_YCR = O_Y + 16 * TH, O_YRT = O_Y + 32 * TH, O_YRB = O_YRT + RW;
    static constexpr int O_CRN = O_YRB + RW;              // 8 corner label slots of 128 bytes
    static_assert(O_CRN + 8 * 128 <= STAGE, "ring boxes fit the y2 / label area");
    static constexpr int STAGES = STAGES_;
    static constexpr int SMEM = STAGES * STAGE + 128;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// Blocking wait: the suspend-time hint lets the warp sleep in hardware until
// the phase flips instead of spinning (a spinning warp steals issue slots from
// the warps that compute).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

template <int TW, int TH>
__device__ __forceinline__ void tma_issue_tile(const Lat2 &L, const TmaMaps &M, uint8_t *stage,
                                               uint64_t *bar, int by, int bx, int tile, int cur,
                                               bool solved) {
    using C = TmaCfg<TW, TH, TW * TH / 4>;   // box geometry does not depend on NT / STAGES
    const int x0 = bx * TW;                       // uniform tiling: lo = index * width
    const int y0 = by * L.ay.base + tile * C::TH;
    // y2 / label maps start at the ghost row above the shard: +1 row
    if (solved) {
        mbar_expect_tx(bar, C::TX);
        tma_load_2d(stage + C::O_A, &M.a, bar, x0, y0);
        tma_load_2d(stage + C::O_Y, &M.y[cur], bar, x0, y0 + 1);
        tma_load_2d(stage + C::O_YR, &M.yr[cur], bar, x0 + TW, y0 + 1);
        tma_load_2d(stage + C::O_H, &M.yhat, bar, x0 - 16, y0);
    } else {
        // out-of-range boxes (grid edges) are zero-filled and still counted
        mbar_expect_tx(bar, C::TX_CLEAN);
        tma_load_2d(stage + C::O_Y, &M.y[cur], bar, x0, y0 + 1);
        tma_load_2d(stage + C::O_YR, &M.yr[cur], bar, x0 + TW, y0 + 1);
        tma_load_2d(stage + C::O_HUP, &M.hrow, bar, x0, y0);
        tma_load_2d(stage + C::O_HDN, &M.hrow, bar, x0, y0 + C::TH + 1);
        tma_load_2d(stage + C::O_HL, &M.hcol, bar, x0 - 16, y0 + 1);
        tma_load_2d(stage + C::O_HR, &M.hcol, bar, x0 + TW, y0 + 1);
        tma_load_2d(stage + C::O_AL, &M.acol, bar, x0, y0);
        tma_load_2d(stage + C::O_AR, &M.acol, bar, x0 + TW - 8, y0);
        tma_load_2d(stage + C::O_AT, &M.arow, bar, x0, y0);
        tma_load_2d(stage + C::O_AB, &M.arow, bar, x0, y0 + C::TH - 1);
    }
}

// Ring-only tile: only the data of the ring groups a re-solved neighbour can
// move.  ld: sides whose ring quads are loaded (1 L, 2 R, 4 U, 8 D); crn:
// corners whose labels across both sides are loaded (1 TL, 2 TR, 4 BL, 8 BR).
template <int TW, int TH>
__device__ __forceinline__ void tma_issue_ring(const Lat2 &L, const TmaMaps &M, uint8_t *stage,
                                               uint64_t *bar, int by, int bx, int tile, int cur,
                                               uint32_t ld, uint32_t crn) {
    using C = TmaCfg<TW, TH, TW * TH / 4>;
    const int x0 = bx * TW;
    const int y0 = by * L.ay.base + tile * C::TH;
    uint32_t tx = 0;
    if (ld & 1u) tx += 48 * TH;
    if (ld & 2u) tx += 48 * TH;
    if (ld & 4u) tx += 4 * TW;
    if (ld & 8u) tx += 4 * TW;
    tx += 32u * (uint32_t)__popc(crn);
    mbar_expect_tx(bar, tx);
    if (ld & 1u) {
        tma_load_2d(stage + C::O_HL, &M.hcol, bar, x0 - 16, y0 + 1);
        tma_load_2d(stage + C::O_AL, &M.acol, bar, x0, y0);
        tma_load_2d(stage + C::O_YCL, &M.yr[cur], bar, x0, y0 + 1);
    }
    if (ld & 2u) {
        tma_load_2d(stage + C::O_HR, &M.hcol, bar, x0 + TW, y0 + 1);
        tma_load_2d(stage + C::O_AR, &M.acol, bar, x0 + TW - 8, y0);
        tma_load_2d(stage + C::O_YCR, &M.yr[cur], bar, x0 + TW - 16, y0 + 1);
    }
    if (ld & 4u) {
        tma_load_2d(stage + C::O_HUP, &M.hrow, bar, x0, y0);
        tma_load_2d(stage + C::O_AT, &M.arow, bar, x0, y0);
        tma_load_2d(stage + C::O_YRT, &M.yrow[cur], bar, x0, y0 + 1);
    }
    if (ld & 8u) {
        tma_load_2d(stage + C::O_HDN, &M.hrow, bar, x0, y0 + C::TH + 1);
        tma_load_2d(stage + C::O_AB, &M.arow, bar, x0, y0 + C::TH - 1);
        tma_load_2d(stage + C::O_YRB, &M.yrow[cur], bar, x0, y0 + C::TH);
    }
    // corner slots: [side label 16 B][label row across the top / bottom 16 B]
    if (crn & 1u) {
        tma_load_2d(stage + C::O_CRN + 0 * 128, &M.h16, bar, x0 - 16, y0 + 1);
        tma_load_2d(stage + C::O_CRN + 1 * 128, &M.h16, bar, x0, y0);
    }
    if (crn & 2u) {
        tma_load_2d(stage + C::O_CRN + 2 * 128, &M.h16, bar, x0 + TW, y0 + 1);
        tma_load_2d(stage + C::O_CRN + 3 * 128, &M.h16, bar, x0 + TW - 16, y0);
    }
    if (crn & 4u) {
        tma_load_2d(stage + C::O_CRN + 4 * 128, &M.h16, bar, x0 - 16, y0 + C::TH);
        tma_load_2d(stage + C::O_CRN + 5 * 128, &M.h16, bar, x0, y0 + C::TH + 1);
    }
    if (crn & 8u) {
        tma_load_2d(stage + C::O_CRN + 6 * 128, &M.h16, bar, x0 + TW, y0 + C::TH);
        tma_load_2d(stage + C::O_CRN + 7 * 128, &M.h16, bar, x0 + TW - 16, y0 + C::TH + 1);
    }
}

// 4 bytes (each 0 or 1) -> 4 bits
__device__ __forceinline__ uint32_t bits_b01(uint32_t w) { return ((w * 0x01020408u) >> 24) & 0xFu; }
// 4 bits -> 4 bytes (each 0 or 1)
__device__ __forceinline__ uint32_t bytes_b01(uint32_t b) { return (b * 0x00204081u) & 0x01010101u; }

// One quad (4 consecutive pixels of a row) of the consensus update.
//   h4  : labels (bytes 0/1)         a2  : multipliers (int16 x 4)
//   cnt : per-pixel count of cross-block neighbours (bytes)
//   nb  : per-pixel sum of their labels (bytes)
// y = clamp(h + a - q * sx) with sx = cnt*h - nb (the solve_global stencil,
// admm.py:136-180); sx enters biased by 4 so the bytewise subtraction never
// borrows.  Returns the new y as bits; writes the new multipliers.
__device__ __forceinline__ uint32_t quad_update(uint32_t h4, uint2 a2, uint32_t cnt, uint32_t nb, int q,
                                                int q4, uint2 &an, uint32_t &clp) {
    const uint32_t sb = ((cnt & (h4 * 0xFFu)) | 0x04040404u) - nb;   // bytes: sx + 4
    const int a0 = (int)__byte_perm(a2.x, 0, 0x9910), a1 = (int)a2.x >> 16;
    const int a3_ = (int)a2.y >> 16, a2_ = (int)__byte_perm(a2.y, 0, 0x9910);
    const int h0 = __byte_perm(h4, 0, 0x4440), h1 = __byte_perm(h4, 0, 0x4441);
    const int h2 = __byte_perm(h4, 0, 0x4442), h3 = __byte_perm(h4, 0, 0x4443);
    const int p0 = a0 + h0 + q4 - q * (int)__byte_perm(sb, 0, 0x4440);
    const int p1 = a1 + h1 + q4 - q * (int)__byte_perm(sb, 0, 0x4441);
    const int p2 = a2_ + h2 + q4 - q * (int)__byte_perm(sb, 0, 0x4442);
    const int p3 = a3_ + h3 + q4 - q * (int)__byte_perm(sb, 0, 0x4443);
    clp |= (uint32_t)(p0 | p1) | (uint32_t)(p2 | p3);   // all in {0,1} <=> OR <= 1
    const int y0 = p0 > 0, y1 = p1 > 0, y2 = p2 > 0, y3 = p3 > 0;
    an.x = __byte_perm((uint32_t)(a0 + h0 - y0), (uint32_t)(a1 + h1 - y1), 0x5410);
    an.y = __byte_perm((uint32_t)(a2_ + h2 - y2), (uint32_t)(a3_ + h3 - y3), 0x5410);
    return (uint32_t)(y0 | (y1 << 1) | (y2 << 2) | (y3 << 3));
}

__device__ __forceinline__ uint32_t lanemask_lt_() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Stage descriptor written by the producer before it arms the stage's barrier
// (the arrive has release semantics; consumers read it after the wait).
struct StageInfo {
    int k;          // block id, or -1: no more work
    int tile;       // tile index within the block
    int flags;      // bit0 re-solved this iteration, bit1 interior clamp memo, bit2 last tile,
                    // bits 3-6 neighbour across L / R / U / D re-solved this iteration,
                    // bits 8-15 ring-group clamp memos (see ring_group),
                    // bit16 ring-only tile, bits 17-20 its loaded sides (L R U D)
    int pad_;
    long long em;   // ring-only: the block's energy partial (it repeats)
};

// Per-block metadata the producer warp gathers for its next 32 blocks
// (lane j: block j), so lane 0 never waits on these loads one block at a time.
struct BlockMeta {
    int k;
    int flags;      // StageInfo flags bits 0-1, 3-6, 8-15
    int mode;       // 0 full tile pass, 1 ring-only, 2 nothing to do (partials repeat)
    int pad_;
    long long em;
};

// Ring groups of a block's boundary quads (clamp memos, part_flags bits
// 8-15): 0 left edge, 1 right edge, 2 top edge, 3 bottom edge, 4-7 corners
// TL TR BL BR; -1 = interior.  A group of a clean block can only move when a
// neighbour across one of its sides was re-solved this iteration.
__device__ __forceinline__ int ring_group(bool lft, bool rgt, bool top, bool bot) {
    if (top) return lft ? 4 : (rgt ? 5 : 2);
    if (bot) return lft ? 6 : (rgt ? 7 : 3);
    if (lft) return 0;
    if (rgt) return 1;
    return -1;
}

// groups touching the re-solved sides (side bits: 1 L, 2 R, 4 U, 8 D)
__device__ __forceinline__ uint32_t active_groups(uint32_t sides) {
    const uint32_t L = sides & 1u, R = (sides >> 1) & 1u, U = (sides >> 2) & 1u, D = (sides >> 3) & 1u;
    return L | (R << 1) | (U << 2) | (D << 3) | ((L | U) << 4) | ((R | U) << 5) | ((L | D) << 6) | ((R | D) << 7);
}

// the pass's diagnostics slots: after K1's per-block ones in overlap mode
// (both kernels are live at once)
__device__ __forceinline__ int64_t *k2_timeline(const Lat2 &L) {
    return L.timeline + (L.ovl ? 8 * (size_t)L.K : 0);
}

// diagnostics (timeline mode, K >= 5 * CTAs): per CTA and stage n < 8,
// [issue, data arrived (warp 0), consumed (warp 0), tile loop done (warp 0)]
// globaltimer stamps after
// the 8 per-CTA slots
__device__ __forceinline__ void stage_stamp(const Lat2 &L, int n, int which) {
    if (!L.timeline || n >= 8 || L.K < 5 * (int)gridDim.x) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    k2_timeline(L)[8 * gridDim.x + (blockIdx.x * 8 + n) * 4 + which] = (int64_t)t;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised: NT consumer threads compute, one producer warp (lane 0)
// claims blocks, issues the TMA loads, and drains each finished block's
// partials -- consumers never wait on a CTA-wide barrier, only on their
// stage's "full" mbarrier; the producer waits on the stage's "empty" one.
// Block scheduling is static round-robin (a pass-wide claim counter was
// measured slower).  Every pass-wide aggregate is an exact integer (the
// residual sum included, see rsq_excess), so results do not depend on which
// CTA took a block.
template <int TW, int TH_, int NT_, int STAGES_>
#ifndef K2T_CPS
#define K2T_CPS 4
#endif
__global__ void __launch_bounds__(NT_ + 32, (NT_ <= 128 ? K2T_CPS : (NT_ <= 256 ? 2 : 1)))
    k_consensus_tma(Lat2 L, const __grid_constant__ TmaMaps M, uint32_t kx_magic, int settle) {
    using C = TmaCfg<TW, TH_, NT_, STAGES_>;
    constexpr int TH = C::TH, NT = C::NT, QPT = C::QPT, QR = TW / 4, LQ = (TW == 64) ? 4 : 5;
    constexpr int ST = C::STAGES;
    extern __shared__ __align__(128) uint8_t smem_t[];
    // keep the shared address space visible to the compiler (LDS, not generic LD)
    uint8_t *base = smem_t + ((128u - (smem_u32(smem_t) & 127u)) & 127u);
    __shared__ __align__(8) uint64_t full[ST], empty[ST];
    __shared__ StageInfo sinfo[ST];
    // per-stage block accumulators (filled at a block's last tile, drained by
    // the producer before the stage is refilled)
    __shared__ unsigned long long accU[ST];
    __shared__ unsigned int accE[ST], accS[ST], accF[ST];

    dope_run_state *st = L.st;
    const int tid = threadIdx.x, lane = tid & 31;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&M.y[0])) : "memory");
    if (L.pdl) {
        griddep_wait();     // K1's labels and solve epochs (PDL launch)
        griddep_launch();   // every CTA is resident: the next K1 may launch and wait
    }
    if (st->stop) return;
    const int cur = st->ycur, best = st->ybest, out = other_buffer(cur, best);
    const int iter = st->iteration;
    ystore_t *__restrict__ y_out = L.y2[out];
    astore_t *a_out = L.a;   // in place
    const bool want_e = iter >= 1;
    const int32_t W = L.W, H = L.ay.dim, q = L.q, BH = L.ay.base, KX = L.ax.k, K = L.K;
    const int q4 = 4 * q;
    const int tpb = BH / TH;                          // tiles per block

    if (tid == NT) {
        if (L.timeline) {   // diagnostics: CTA start (slot 6 of entry blockIdx)
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            k2_timeline(L)[8 * blockIdx.x + 6] = (int64_t)t;
        }
        for (int i = 0; i < ST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NT / 32);
            accU[i] = 0;
            accE[i] = 0;
            accS[i] = 0;
            accF[i] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= NT) {
        // ================= producer warp =================
        // All 32 lanes gather the metadata of the CTA's next 32 blocks (static
        // round-robin assignment) and settle the blocks with nothing to do;
        // lane 0 then issues the TMA loads and drains the finished stages.
        const int plane = tid - NT;
        __shared__ BlockMeta meta[32];
        const int KY = K / KX;
        const uint32_t ep_now = (uint32_t)(iter + 1);
        // phase A: this iteration's solved blocks, dealt out evenly from K1's
        // list (they carry the full tile work); phase B: every other block,
        // static round-robin (clean blocks: mostly ring-only or settled)
        const int G = (int)gridDim.x, bid = (int)blockIdx.x;
        // (a CTA with at most two blocks has nothing to balance: skip phase A
        // and the dependent list read it costs)
        const int nsolved = (L.skip_clean && L.slist && K > 2 * G) ? solved_count(L) : 0;
        const int nA = bid < nsolved ? (nsolved - 1 - bid) / G + 1 : 0;
        const int nmine = nA + (bid < K ? (K - 1 - bid) / G + 1 : 0);
        CtaAgg agg;   // this CTA's pass aggregates (exact integers), lane 0
        // Draining a stage is split: `take` reads the stage's descriptor and
        // accumulators (shared memory) and resets them before the stage is
        // refilled; `finish` then does the global writes -- per-block
        // partials, stamps and the dirty marks -- while the refill's TMA loads
        // are in flight.  The marks' atomics go out together, not one round
        // trip after another (they used to stall the producer ~3 us per
        // re-solved block).
        struct Taken {
            StageInfo info;
            unsigned long long u;
            unsigned int e, sq, f;
        };
        auto take = [&](int s, Taken &t) {
            t.info = sinfo[s];
            if (!(t.info.flags & 4)) return false;
            t.e = accE[s];
            t.u = accU[s];
            t.sq = accS[s];
            t.f = accF[s];
            accE[s] = 0;
            accS[s] = 0;
            accF[s] = 0;
            accU[s] = 0;
            return true;
        };
        uint32_t *const next_list = L.dlist ? dirty_list(L, iter + 1) : nullptr;
        // Worklist marks, software-pipelined over the CTA's drains so the
        // producer never waits on an atomic's return value: a drain issues
        // the exchanges of its block's marks (first marks join the worklist),
        // turns the previous drain's exchange results into one slot
        // reservation, and writes the entries of the reservation before that.
        int p1k[5], p2k[5];
        uint32_t p1old[5], p1m = 0u, p2new = 0u, p2slot = 0u;
        auto mark_pipe = [&](const int (&kk)[5], uint32_t mm) {
            if (p2new) {   // stage 3: entries of the reservation issued two drains ago
                uint32_t slot = p2slot;
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    if (p2new >> i & 1u) {
                        if (slot < (uint32_t)K) next_list[1 + slot] = (uint32_t)p2k[i];
                        ++slot;
                    }
                p2new = 0u;
            }
            if (p1m) {     // stage 2: reserve slots for the first marks of the last drain
                uint32_t nm = 0u;
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    if ((p1m >> i & 1u) && p1old[i] == 0u) nm |= 1u << i;
                if (nm) {
                    p2slot = atomicAdd(next_list, (uint32_t)__popc(nm));
                    p2new = nm;
#pragma unroll
                    for (int i = 0; i < 5; ++i) p2k[i] = p1k[i];
                }
                p1m = 0u;
            }
            if (mm) {      // stage 1: the exchanges of this drain
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    p1k[i] = kk[i];
                    p1old[i] = (mm >> i & 1u) ? atomicExch(&L.dirty[kk[i]], 1u) : 1u;
                }
                p1m = mm;
            }
        };
        auto finish = [&](const Taken &t) {
            const StageInfo &info = t.info;
            const int k = info.k;
            const bool ring = (info.flags & 0x10000) != 0;
            const int64_t e = ring ? (int64_t)info.em : (int64_t)L.lamw * t.e;
            const int64_t u2 = (int64_t)t.u;
            const int64_t sq = t.sq;
            const unsigned f = t.f;
            const bool solved = info.flags & 1;
            const bool memo = solved ? (f & 64u) != 0 : (info.flags & 2) != 0;
            // ring groups: recomputed ones take this pass's clamp bits, the
            // others (clean block, no re-solved neighbour on their sides) keep
            // their memo
            const uint32_t fresh = (f >> 8) & 0xFFu;
            const uint32_t act = solved ? 0xFFu : active_groups((uint32_t)(info.flags >> 3) & 0xFu);
            const uint32_t gbits = (fresh & act) | (((uint32_t)info.flags >> 8) & 0xFFu & ~act);
            const int clamped = (gbits || memo) ? 1 : 0;
            L.pe[k] = e;
            L.pu[k] = u2;
            L.pr[k] = sq;
            L.pf[k] = clamped | (memo ? 64 : 0) | (int)(gbits << 8);
            agg.add_block(e, u2, sq, clamped);
            // dirty marks for the next iteration: self, L, R, U, D
            const int kk[5] = {k, k - 1, k + 1, k - KX, k + KX};
            const uint32_t mm = ((f >> 1) & 7u) | ((f & 16u) && k - KX >= 0 ? 8u : 0u) |
                                ((f & 32u) && k + KX < K ? 16u : 0u);
            if (!next_list) {
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    if (mm >> i & 1u) L.dirty[kk[i]] = 1u;
            } else {
                mark_pipe(kk, mm);
            }
            // the output buffer now holds the block's whole iterate
            ybuf_stamp(L, out)[k] = ep_now;
            if (want_e) pe_stamp(L)[k] = ep_now;
            if (f & 128u) ychg_stamp(L)[k] = ep_now;
        };
        auto drain = [&](int s) {
            Taken t;
            if (take(s, t)) finish(t);
        };
        int n = 0;   // stages issued (lane 0)
        // Queue mode (the TMA pass with a solved list): phase B's blocks with
        // tile work (clean full passes, ring-only) go to a pass-wide queue
        // (L.kq) that every CTA drains once its own phase-A / phase-B work is
        // issued, so the stage chain of a CTA no longer depends on how many
        // such blocks its static share held (measured: 1..7 stages per CTA).
        const bool qmode = L.kq != nullptr;
        // overlap mode: a block whose labels (or a re-solved neighbour's) K1
        // has not published yet is deferred behind the CTA's ready blocks,
        // then awaited in order
        auto ready = [&](const BlockMeta &bm) {
            const uint32_t sd = ((uint32_t)bm.flags >> 3) & 0xFu;
            const uint32_t *kd = L.kdone;
            bool r = !(bm.flags & 1) || ld_acquire_gpu(kd + bm.k) == ep_now;
            if (r && (sd & 1u)) r = ld_acquire_gpu(kd + bm.k - 1) == ep_now;
            if (r && (sd & 2u)) r = ld_acquire_gpu(kd + bm.k + 1) == ep_now;
            if (r && (sd & 4u)) r = ld_acquire_gpu(kd + bm.k - KX) == ep_now;
            if (r && (sd & 8u)) r = ld_acquire_gpu(kd + bm.k + KX) == ep_now;
            return r;
        };
        // the stages of one block (lane 0)
        auto issue_block = [&](const BlockMeta &bm) {
            const int by = (int)__umulhi((uint32_t)bm.k, kx_magic), bx = bm.k - by * KX;
            const bool hl = bx > 0, hr = bx + 1 < KX, hu = by > 0 || L.gup, hd = by + 1 < KY || L.gdn;
            const uint32_t sd = ((uint32_t)bm.flags >> 3) & 0xFu;
            for (int tile = 0; tile < tpb; ++tile) {
                const int s = n % ST;
                Taken pend;
                bool has_pend = false;
                if (n >= ST) {
                    mbar_wait(&empty[s], ((n / ST) - 1) & 1);
                    has_pend = take(s, pend);
                }
                int fl = bm.flags | (tile == tpb - 1 ? 4 : 0);
                uint8_t *stg = base + s * C::STAGE;
                sinfo[s].k = bm.k;
                sinfo[s].tile = tile;
                sinfo[s].em = bm.em;
                if (bm.mode == 1) {
                    const bool tt = tile == 0, tb = tile == tpb - 1;
                    const uint32_t ld = (sd & 3u) | (tt ? sd & 4u : 0u) | (tb ? sd & 8u : 0u);
                    uint32_t crn = 0;
                    if (tt && hu && hl && (sd & 5u)) crn |= 1u;
                    if (tt && hu && hr && (sd & 6u)) crn |= 2u;
                    if (tb && hd && hl && (sd & 9u)) crn |= 4u;
                    if (tb && hd && hr && (sd & 10u)) crn |= 8u;
                    sinfo[s].flags = fl | 0x10000 | (int)(ld << 17);
                    stage_stamp(L, n, 0);
                    tma_issue_ring<TW, TH>(L, M, stg, &full[s], by, bx, tile, cur, ld, crn);
                } else {
                    sinfo[s].flags = fl;
                    stage_stamp(L, n, 0);
                    tma_issue_tile<TW, TH>(L, M, stg, &full[s], by, bx, tile, cur, fl & 1);
                }
                if (has_pend) finish(pend);   // while the refill is in flight
                ++n;
            }
        };
        for (int c0 = 0; c0 < nmine; c0 += 32) {
            const int nc = nmine - c0 < 32 ? nmine - c0 : 32;
            int64_t eskip = 0;
            int fskip = 0, nskip = 0;
            bool qpush = false, qmode1 = false;
            if (plane < nc) {
                const int j = c0 + plane;
                const bool isA = j < nA;
                const int aslot = bid + j * G;
                const int kk = isA ? (int)solved_list(L)[aslot] : bid + (j - nA) * G;
                const int by = (int)__umulhi((uint32_t)kk, kx_magic), bx = kk - by * KX;
                // every load of this block's metadata in one independent
                // round (neighbour indices clamped in range, results masked)
                const int kl = bx > 0 ? kk - 1 : kk, kr = bx + 1 < KX ? kk + 1 : kk;
                const int ku = by > 0 ? kk - KX : kk, kd = by + 1 < KY ? kk + KX : kk;
                const uint32_t *ych = ychg_stamp(L);
                const uint32_t epk = __ldcg(L.dirty + K + kk);
                const int memo = __ldcg(L.pf + kk);
                const uint32_t el = __ldcg(L.dirty + K + kl), er = __ldcg(L.dirty + K + kr);
                const uint32_t eu = __ldcg(L.dirty + K + ku), ed = __ldcg(L.dirty + K + kd);
                const uint32_t ps = __ldcg(pe_stamp(L) + kk), yk = __ldcg(ych + kk);
                const uint32_t so = __ldcg(ybuf_stamp(L, out) + kk);
                const uint32_t sl = __ldcg(solved_slot(L) + kk);
                const long long pek = __ldcg(reinterpret_cast<const long long *>(L.pe) + kk);
                // neighbours re-solved this iteration (L R U D bits; a ghost
                // row from another shard is always treated as moved)
                uint32_t sd = 0;
                if (bx > 0 && el == ep_now) sd |= 1u;
                if (bx + 1 < KX && er == ep_now) sd |= 2u;
                if (by > 0 ? eu == ep_now : L.gup != 0) sd |= 4u;
                if (by + 1 < KY ? ed == ep_now : L.gdn != 0) sd |= 8u;
                const bool solved = !L.skip_clean || epk == ep_now;
                // mode 3: nothing here -- a phase-A entry that is not its
                // block's latest slot, or a solved block phase A deals with
                int mode = 0;
                if (isA) {
                    if (!solved || sl != (uint32_t)aslot + 1u) mode = 3;
                } else if (L.skip_clean && solved) {
                    // a block K1 solved this iteration sits in the solved list
                    // exactly once (phase A): its slot is this iteration's
                    if (nsolved > 0 ? (sl >= 1u && sl <= (uint32_t)nsolved) : false) mode = 3;
                }
                long long em = 0;
                // clean block: neither it nor the facing pixels
                // of its right / lower neighbour (the other ends of its pairs)
                // moved in the last pass -- a move there would have marked it
                // dirty -- so its energy partial repeats when the last pass
                // stored one (energy stamp); the output buffer already holds
                // its iterate when it received it after the block's last change
                const uint32_t it32 = (uint32_t)iter;
                const bool ok = mode == 0 && !solved && iter >= 2 && settle && ps == it32 && so != 0u && so >= yk;
                if (ok) {
                    em = pek;
                    mode = sd ? 1 : 2;
                }
                if (mode == 2) {
                    // every quad is a fixed point: partials, flags and the
                    // output buffer's copy all repeat
                    L.pu[kk] = 0;
                    L.pr[kk] = 0;
                    ybuf_stamp(L, out)[kk] = ep_now;
                    pe_stamp(L)[kk] = ep_now;
                    eskip = em;
                    fskip = memo & 1;
                    nskip = 1;
                }
                meta[plane].k = kk;
                meta[plane].flags = (solved ? 1 : 0) | ((memo & 64) ? 2 : 0) | (int)(sd << 3) | (memo & 0xFF00);
                // queue mode: a phase-B block with tile work joins the pass's
                // queue (any CTA may take it) instead of this CTA's stages
                qpush = qmode && !isA && mode <= 1;
                qmode1 = mode == 1;
                meta[plane].mode = qpush ? 3 : mode;
                meta[plane].em = em;
            }
            // queue mode: this batch's appends, reserved now (lane 0), written
            // once the CTA's own stages are issued
            uint32_t qm = 0u, qslot = 0u;
            if (qmode) {
                qm = __ballot_sync(FULLMASK, qpush);
                if (qm && plane == 0) qslot = atomicAdd(L.kq + 4 * (size_t)K, (uint32_t)__popc(qm));
            }
            // fold the settled blocks into lane 0's aggregates
            eskip = warp_sum(eskip);
            fskip = __reduce_or_sync(FULLMASK, fskip);
            nskip = __reduce_add_sync(FULLMASK, nskip);
            __syncwarp();
            if (plane == 0 && c0 == 0 && L.timeline) {   // diagnostics: metadata gathered (slot 0)
                uint64_t t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                k2_timeline(L)[8 * blockIdx.x + 0] = (int64_t)t;
            }
            if (plane == 0) {
                if (nskip) {
                    agg.E += eskip;
                    agg.F |= fskip;
                    agg.M = agg.M > 0 ? agg.M : 0;
                }
                uint32_t deferred = 0;
                for (int pass = 0; pass < (L.ovl ? 2 : 1); ++pass)
                for (int j = 0; j < nc; ++j) {
                    const BlockMeta bm = meta[j];
                    if (bm.mode >= 2) continue;
                    if (L.ovl) {
                        if (pass == 0 && !ready(bm)) {
                            deferred |= 1u << j;
                            continue;
                        }
                        if (pass == 1) {
                            if (!(deferred >> j & 1u)) continue;
                            while (!ready(bm)) __nanosleep(128);
                        }
                        // labels written by other CTAs (generic proxy) before the TMA reads them
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    issue_block(bm);
                }
            }
            __syncwarp();
            if (qm) {   // warp-aggregated append: entry = {k + 1, flags | mode << 29, em}
                const uint32_t slot = __shfl_sync(FULLMASK, qslot, 0) + __popc(qm & lanemask_lt_());
                if (qpush) {
                    const BlockMeta &bm = meta[plane];
                    uint32_t *e = L.kq + 4 * (size_t)slot;
                    e[1] = (uint32_t)bm.flags | (qmode1 ? (1u << 29) : 0u);
                    e[2] = (uint32_t)(unsigned long long)bm.em;
                    e[3] = (uint32_t)((unsigned long long)bm.em >> 32);
                    st_release_gpu(e, (uint32_t)bm.k + 1u);
                }
                __syncwarp();
            }
        }
        if (qmode) {
            // this CTA's appends are out: count it done, then take queue
            // entries until every CTA is done and the queue is exhausted
            uint32_t *qlen = L.kq + 4 * (size_t)K, *qclaim = qlen + 1, *qdone = qlen + 2;
            if (plane == 0) {
                __threadfence();
                atomicAdd(qdone, 1u);
                for (;;) {
                    const uint32_t idx = atomicAdd(qclaim, 1u);
                    uint32_t *e = L.kq + 4 * (size_t)idx;
                    uint32_t k1 = 0;
                    for (;;) {
                        if (idx < (uint32_t)K) k1 = ld_acquire_gpu(e);
                        if (k1) break;
                        if (ld_acquire_gpu(qdone) == (uint32_t)G && idx >= ld_acquire_gpu(qlen)) break;
                        __nanosleep(64);
                    }
                    if (!k1) break;
                    BlockMeta bm;
                    bm.k = (int)k1 - 1;
                    const uint32_t fw = __ldcg(e + 1);
                    bm.flags = (int)(fw & ~(1u << 29));
                    bm.mode = (fw >> 29) & 1u;
                    bm.em = (long long)(((unsigned long long)__ldcg(e + 3) << 32) | __ldcg(e + 2));
                    e[0] = 0u;   // consumed (the queue is empty again when the pass ends)
                    if (L.ovl) {
                        while (!ready(bm)) __nanosleep(128);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    issue_block(bm);
                }
            }
            __syncwarp();
        }
        if (plane != 0) return;
        if (L.timeline) {   // diagnostics: last stage issued (slot 1), stages (slot 4), phase-A blocks (slot 5)
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            k2_timeline(L)[8 * blockIdx.x + 1] = (int64_t)t;
            k2_timeline(L)[8 * blockIdx.x + 4] = n;
            k2_timeline(L)[8 * blockIdx.x + 5] = nA;
        }
        {   // end marker
            const int s = n % ST;
            if (n >= ST) {
                mbar_wait(&empty[s], ((n / ST) - 1) & 1);
                drain(s);
            }
            sinfo[s].k = -1;
            mbar_arrive(&full[s]);
        }
        // drain the stages still in flight when the end marker went out
        for (int m = (n - ST + 1 > 0 ? n - ST + 1 : 0); m < n; ++m) {
            const int s = m % ST;
            mbar_wait(&empty[s], (m / ST) & 1);
            drain(s);
        }
        if (next_list) {   // flush the mark pipeline
            const int none[5] = {0, 0, 0, 0, 0};
            mark_pipe(none, 0u);
            mark_pipe(none, 0u);
        }
        if (L.timeline) {   // diagnostics: CTA end (slot 7)
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            k2_timeline(L)[8 * blockIdx.x + 7] = (int64_t)t;
        }
        if (L.timeline) {   // diagnostics: stages drained (slot 2)
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            k2_timeline(L)[8 * blockIdx.x + 2] = (int64_t)t;
        }
        pass_tail(L, agg, cur, best, out);
        return;
    }

    // ================= consumer warps =================
    int rr_[QPT], c0_[QPT];
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int t = tid + j * NT;
        rr_[j] = t >> LQ;
        c0_[j] = (t & (QR - 1)) << 2;
    }
    int64_t du = 0;
    int ss = 0, quad_acc = 0;
    // fl: bit1 self, bit2 left, bit3 right, bit4 up, bit5 down
    // gcl: ring-group clamp bits; clpi: OR of the interior quads' pre-clamp values
    uint32_t fl = 0, gcl = 0, clpi = 0;
    for (int n = 0;; ++n) {
        const int s = n % ST;
        mbar_wait(&full[s], (n / ST) & 1);
        if (tid == 0) stage_stamp(L, n, 1);
        const StageInfo info = sinfo[s];
        if (info.k < 0) break;
        const int k = info.k, tile = info.tile;
        const bool solved = info.flags & 1;
        const int by = (int)__umulhi((uint32_t)k, kx_magic), bx = k - by * KX;
        const int lo_r = by * BH, lo_c = bx * TW;
        const bool has_up = lo_r > 0 || L.gup, has_dn = lo_r + BH < H || L.gdn, has_lf = lo_c > 0,
                   has_rt = lo_c + TW < W;
        const bool last_row_pairs = lo_r + BH < H || L.gdn;   // pairs below the block's last row
        {
            const uint8_t *sb = base + s * C::STAGE;
            const astore_t *sa = reinterpret_cast<const astore_t *>(sb + C::O_A);
            const uint8_t *sy = sb + C::O_Y;
            const uint8_t *syr = sb + C::O_YR;
            const uint8_t *sh = sb + C::O_H + C::YHW + 16;      // label of tile pixel (0,0)
            const int r0 = tile * TH;
            const int64_t gt = (int64_t)(lo_r + r0) * W + lo_c;   // global index of tile (0,0)
            // E(y_{t-1}) pair terms of one quad: bytes are 0/2, so each
            // differing pair is exactly one set bit of the XOR (all lanes call
            // this together: the right neighbour comes from the next lane)
            auto pair_energy = [&](int rr, int c0, uint32_t yo) {
                const uint32_t nxt = __shfl_down_sync(FULLMASK, yo, 1);
                uint32_t rw = nxt;
                if (c0 + 4 == TW) rw = has_rt ? (uint32_t)syr[rr * 16] : (yo >> 24);
                const uint32_t yb = (r0 + rr + 1 < BH || last_row_pairs)
                                        ? *reinterpret_cast<const uint32_t *>(sy + (rr + 1) * TW + c0)
                                        : yo;
                quad_acc += __popc(yo ^ __funnelshift_r(yo, rw, 8)) + __popc(yo ^ yb);
            };
            // consensus update of one quad given its multipliers, own labels
            // and cross-block neighbour labels (count / sum per pixel)
            // running unary term u * (y2_new - y2_old) of one quad
            auto unary = [&](int64_t G, uint32_t yw, uint32_t yo) {
                const int4 uv = __ldg(reinterpret_cast<const int4 *>(L.u + G));
                du += (int64_t)uv.x * ((int)(yw & 0xFFu) - (int)(yo & 0xFFu)) +
                      (int64_t)uv.y * ((int)((yw >> 8) & 0xFFu) - (int)((yo >> 8) & 0xFFu)) +
                      (int64_t)uv.z * ((int)((yw >> 16) & 0xFFu) - (int)((yo >> 16) & 0xFFu)) +
                      (int64_t)uv.w * ((int)(yw >> 24) - (int)(yo >> 24));
            };
            // defer: 0 = gather u now (ring quads), else the caller batches it
            auto update = [&](int rr, int c0, uint32_t yo, uint32_t h4, uint2 av, uint32_t cnt, uint32_t nb,
                              bool lft, bool rgt, bool top, bool bot, int grp, uint32_t *yw_out = nullptr) {
                const int64_t G = gt + (int64_t)rr * W + c0;
                uint2 an;
                uint32_t cq = 0;
                const uint32_t yn = quad_update(h4, av, cnt, nb, q, q4, an, cq);
                if (grp >= 0) gcl |= (cq > 1u ? 1u : 0u) << grp;
                else clpi |= cq;
                const uint32_t hb = bits_b01(h4);
                ss += __popc(hb ^ yn);
                const uint32_t yw = bytes_b01(yn) << 1;            // y2 bytes 0/2
                const uint32_t chg = yw ^ yo;
                fl |= (chg | (hb ^ yn)) ? 2u : 0u;
                fl |= chg ? 128u : 0u;   // the block's iterate moved (ychg stamp)
                __stcs(reinterpret_cast<uint2 *>(a_out + G), an);
                __stcg(reinterpret_cast<unsigned int *>(y_out + G), yw);
                if (yw_out) *yw_out = yw;
                if (chg) {
                    if (!yw_out) unary(G, yw, yo);   // only where y moved
                    const uint32_t em = (lft ? 4u : 0u) | (rgt ? 8u : 0u) | (top ? 16u : 0u) | (bot ? 32u : 0u);
                    const uint32_t mk = 0x30u | ((chg & 0xFFu) ? 4u : 0u) | ((chg >> 24) ? 8u : 0u);
                    fl |= em & mk;
                }
            };
            if (solved) {
                uint32_t ywq[QPT], yoq[QPT];
#pragma unroll
                for (int j = 0; j < QPT; ++j) {
                    const int rr = rr_[j], c0 = c0_[j];
                    const int r = r0 + rr;                         // row within block
                    const uint32_t yo = *reinterpret_cast<const uint32_t *>(sy + rr * TW + c0);
                    if (want_e) pair_energy(rr, c0, yo);
                    const bool lft = (c0 == 0) && has_lf, rgt = (c0 + 4 == TW) && has_rt;
                    const bool top = (r == 0) && has_up, bot = (r == BH - 1) && has_dn;
                    const uint8_t *hrow = sh + rr * C::YHW + c0;
                    const uint2 av = *reinterpret_cast<const uint2 *>(sa + rr * TW + c0);
                    const uint32_t h4 = *reinterpret_cast<const uint32_t *>(hrow);
                    uint32_t cnt = 0, nb = 0;
                    if (top) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(hrow - C::YHW); }
                    if (bot) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(hrow + C::YHW); }
                    if (lft) { cnt += 1u; nb += hrow[-1]; }
                    if (rgt) { cnt += 1u << 24; nb += (uint32_t)hrow[4] << 24; }
                    update(rr, c0, yo, h4, av, cnt, nb, lft, rgt, top, bot, ring_group(lft, rgt, top, bot), &ywq[j]);
                    yoq[j] = yo;
                }
                // the unary term of the quads whose y moved: their u loads
                // all in flight together instead of one latency per quad
                int4 uq[QPT];
#pragma unroll
                for (int j = 0; j < QPT; ++j) {
                    const int64_t G = gt + (int64_t)rr_[j] * W + c0_[j];
                    uq[j] = ywq[j] != yoq[j] ? __ldg(reinterpret_cast<const int4 *>(L.u + G)) : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int j = 0; j < QPT; ++j) {
                    const uint32_t yw = ywq[j], yo = yoq[j];
                    du += (int64_t)uq[j].x * ((int)(yw & 0xFFu) - (int)(yo & 0xFFu)) +
                          (int64_t)uq[j].y * ((int)((yw >> 8) & 0xFFu) - (int)((yo >> 8) & 0xFFu)) +
                          (int64_t)uq[j].z * ((int)((yw >> 16) & 0xFFu) - (int)((yo >> 16) & 0xFFu)) +
                          (int64_t)uq[j].w * ((int)(yw >> 24) - (int)(yo >> 24));
                }
            } else if (info.flags & 0x10000) {
                // ring-only tile: the output buffer already holds the block's
                // iterate and its energy partial repeats, so only the ring
                // groups on the sides whose neighbour was re-solved are
                // recomputed, from the ring boxes the producer loaded
                const bool tile_top = tile == 0 && has_up, tile_bot = tile == tpb - 1 && has_dn;
                const uint32_t act = active_groups((uint32_t)(info.flags >> 3) & 0xFu);
                const uint32_t ld = ((uint32_t)info.flags >> 17) & 0xFu;
                const int nT = tile_top ? QR : 0, nB = tile_bot ? QR : 0;
                const int rlo = tile_top ? 1 : 0, rhi = tile_bot ? TH - 1 : TH;
                const int ncand = nT + nB + 2 * (rhi - rlo);
                for (int i = tid; i < ncand; i += NT) {
                    int rr, c0;
                    if (i < nT) { rr = 0; c0 = 4 * i; }
                    else if (i < nT + nB) { rr = TH - 1; c0 = 4 * (i - nT); }
                    else { const int jj = i - nT - nB; rr = rlo + (jj >> 1); c0 = (jj & 1) ? TW - 4 : 0; }
                    const bool lft = (c0 == 0) && has_lf, rgt = (c0 + 4 == TW) && has_rt;
                    const bool top = rr == 0 && tile_top, bot = rr == TH - 1 && tile_bot;
                    const int grp = ring_group(lft, rgt, top, bot);
                    if (grp < 0 || !((act >> grp) & 1u)) continue;   // fixed point: already in the buffer
                    uint32_t yo;
                    uint2 av;
                    if (lft && (ld & 1u)) {
                        yo = *reinterpret_cast<const uint32_t *>(sb + C::O_YCL + rr * 16);
                        av = *reinterpret_cast<const uint2 *>(sb + C::O_AL + rr * 16);
                    } else if (rgt && (ld & 2u)) {
                        yo = *reinterpret_cast<const uint32_t *>(sb + C::O_YCR + rr * 16 + 12);
                        av = *reinterpret_cast<const uint2 *>(sb + C::O_AR + rr * 16 + 8);
                    } else if (top) {
                        yo = *reinterpret_cast<const uint32_t *>(sb + C::O_YRT + c0);
                        av = *reinterpret_cast<const uint2 *>(sb + C::O_AT + 2 * c0);
                    } else {
                        yo = *reinterpret_cast<const uint32_t *>(sb + C::O_YRB + c0);
                        av = *reinterpret_cast<const uint2 *>(sb + C::O_AB + 2 * c0);
                    }
                    const uint32_t h4 = yo >> 1;                   // own labels == y2 / 2
                    uint32_t cnt = 0, nb = 0;
                    if (top) {
                        cnt += 0x01010101u;
                        nb += lft ? *reinterpret_cast<const uint32_t *>(sb + C::O_CRN + 1 * 128)
                                  : rgt ? *reinterpret_cast<const uint32_t *>(sb + C::O_CRN + 3 * 128 + 12)
                                        : *reinterpret_cast<const uint32_t *>(sb + C::O_HUP + c0);
                    }
                    if (bot) {
                        cnt += 0x01010101u;
                        nb += lft ? *reinterpret_cast<const uint32_t *>(sb + C::O_CRN + 5 * 128)
                                  : rgt ? *reinterpret_cast<const uint32_t *>(sb + C::O_CRN + 7 * 128 + 12)
                                        : *reinterpret_cast<const uint32_t *>(sb + C::O_HDN + c0);
                    }
                    if (lft) {
                        cnt += 1u;
                        nb += top ? sb[C::O_CRN + 0 * 128 + 15] : bot ? sb[C::O_CRN + 4 * 128 + 15] : sb[C::O_HL + rr * 16 + 15];
                    }
                    if (rgt) {
                        cnt += 1u << 24;
                        nb += (uint32_t)(top ? sb[C::O_CRN + 2 * 128] : bot ? sb[C::O_CRN + 6 * 128] : sb[C::O_HR + rr * 16]) << 24;
                    }
                    update(rr, c0, yo, h4, av, cnt, nb, lft, rgt, top, bot, grp);
                }
            } else {
                // clean block: the interior is a fixed point, so the bulk pass
                // only carries y into the rotating buffer (and the energy); the
                // ring quads -- the only ones a neighbour's new labels can move
                // -- are updated in a second pass spread over all threads
                // -- and only on the sides whose neighbour was re-solved.  The
                // bulk pass works on 16-byte chunks (4 quads per thread step).
                const bool tile_top = tile == 0 && has_up, tile_bot = tile == tpb - 1 && has_dn;
                const uint32_t act = active_groups((uint32_t)(info.flags >> 3) & 0xFu);
                constexpr int CPR = TW / 16, NCH = TH * TW / 16;   // chunks per row / per tile
                for (int ci = tid; ci < NCH; ci += NT) {
                    const int rr = ci / CPR, cc = (ci % CPR) * 16;
                    const uint4 yo = *reinterpret_cast<const uint4 *>(sy + rr * TW + cc);
                    if (want_e) {
                        // pairs of the previous iterate: bytes are 0/2, so each
                        // differing pair is one set bit of the XOR
                        const uint32_t nx = __shfl_down_sync(FULLMASK, yo.x, 1);
                        uint32_t rw = nx;
                        if (cc + 16 == TW) rw = has_rt ? (uint32_t)syr[rr * 16] : (yo.w >> 24);
                        const uint4 yb = (r0 + rr + 1 < BH || last_row_pairs)
                                             ? *reinterpret_cast<const uint4 *>(sy + (rr + 1) * TW + cc)
                                             : yo;
                        quad_acc += __popc(yo.x ^ __funnelshift_r(yo.x, yo.y, 8)) +
                                    __popc(yo.y ^ __funnelshift_r(yo.y, yo.z, 8)) +
                                    __popc(yo.z ^ __funnelshift_r(yo.z, yo.w, 8)) +
                                    __popc(yo.w ^ __funnelshift_r(yo.w, rw, 8)) + __popc(yo.x ^ yb.x) +
                                    __popc(yo.y ^ yb.y) + __popc(yo.z ^ yb.z) + __popc(yo.w ^ yb.w);
                    }
                    // carry y into the rotating buffer, except the words of
                    // active ring quads (the ring pass writes those)
                    uint32_t skip = 0;
                    const bool trow = rr == 0 && tile_top, brow = rr == TH - 1 && tile_bot;
                    if (trow || brow) {
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const int c0 = cc + 4 * w;
                            const int grp = ring_group(c0 == 0 && has_lf, c0 + 4 == TW && has_rt, trow, brow);
                            if (grp >= 0 && ((act >> grp) & 1u)) skip |= 1u << w;
                        }
                    } else {
                        if (cc == 0 && has_lf && (act & 1u)) skip |= 1u;
                        if (cc + 16 == TW && has_rt && (act & 2u)) skip |= 8u;
                    }
                    const int64_t G = gt + (int64_t)rr * W + cc;
                    if (!skip) {
                        __stcg(reinterpret_cast<uint4 *>(y_out + G), yo);
                    } else {
                        const uint32_t wv[4] = {yo.x, yo.y, yo.z, yo.w};
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            if (!((skip >> w) & 1u)) __stcg(reinterpret_cast<unsigned int *>(y_out + G) + w, wv[w]);
                    }
                }
                // ring candidates: the block's first / last row when this tile
                // holds it, then the two edge quads of the remaining rows
                const int nT = tile_top ? QR : 0, nB = tile_bot ? QR : 0;
                const int rlo = tile_top ? 1 : 0, rhi = tile_bot ? TH - 1 : TH;
                const int ncand = nT + nB + 2 * (rhi - rlo);
                for (int i = tid; i < ncand; i += NT) {
                    int rr, c0;
                    if (i < nT) { rr = 0; c0 = 4 * i; }
                    else if (i < nT + nB) { rr = TH - 1; c0 = 4 * (i - nT); }
                    else { const int jj = i - nT - nB; rr = rlo + (jj >> 1); c0 = (jj & 1) ? TW - 4 : 0; }
                    const bool lft = (c0 == 0) && has_lf, rgt = (c0 + 4 == TW) && has_rt;
                    const bool top = rr == 0 && tile_top, bot = rr == TH - 1 && tile_bot;
                    const int grp = ring_group(lft, rgt, top, bot);
                    if (grp < 0 || !((act >> grp) & 1u)) continue;   // fixed point: copied by the bulk pass
                    const uint32_t yo = *reinterpret_cast<const uint32_t *>(sy + rr * TW + c0);
                    uint2 av;
                    if (lft) av = *reinterpret_cast<const uint2 *>(sb + C::O_AL + rr * 16);
                    else if (rgt) av = *reinterpret_cast<const uint2 *>(sb + C::O_AR + rr * 16 + 8);
                    else if (top) av = *reinterpret_cast<const uint2 *>(sb + C::O_AT + 2 * c0);
                    else av = *reinterpret_cast<const uint2 *>(sb + C::O_AB + 2 * c0);
                    const uint32_t h4 = yo >> 1;                   // own labels == y2 / 2
                    uint32_t cnt = 0, nb = 0;
                    if (top) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(sb + C::O_HUP + c0); }
                    if (bot) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(sb + C::O_HDN + c0); }
                    if (lft) { cnt += 1u; nb += sb[C::O_HL + rr * 16 + 15]; }
                    if (rgt) { cnt += 1u << 24; nb += (uint32_t)sb[C::O_HR + rr * 16] << 24; }
                    update(rr, c0, yo, h4, av, cnt, nb, lft, rgt, top, bot, grp);
                }
            }
        }
        if (tid == 0) stage_stamp(L, n, 3);
        if (info.flags & 4) {
            // block done in this warp: one shared atomic per quantity
            const unsigned e = __reduce_add_sync(FULLMASK, (unsigned)quad_acc);
            const unsigned sq = __reduce_add_sync(FULLMASK, (unsigned)ss);
            const unsigned f = __reduce_or_sync(FULLMASK, fl | (gcl << 8) | (clpi > 1u ? 64u : 0u));
            int64_t u2 = 0;
            if (__any_sync(FULLMASK, du != 0)) u2 = warp_sum(du);
            if (lane == 0) {
                if (e) atomicAdd(&accE[s], e);
                if (sq) atomicAdd(&accS[s], sq);
                if (f) atomicOr(&accF[s], f);
                if (u2) atomicAdd(&accU[s], (unsigned long long)u2);
            }
            du = 0;
            ss = 0;
            quad_acc = 0;
            fl = 0;
            gcl = 0;
            clpi = 0;
        }
        // this warp is done with stage s
        __syncwarp();
        if (tid == 0) stage_stamp(L, n, 2);
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}
