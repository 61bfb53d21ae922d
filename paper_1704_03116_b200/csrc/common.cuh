// common.cuh -- helpers shared by the lattice kernels (dope_lattice.cu,
// dope_float.cu): block geometry of the reference's partition rule and the
// one-warp bit-parallel global-relabel BFS.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define FULLMASK 0xffffffffu

// Checked builds (-DDOPE_BOUNDS, `python -m paper_1704_03116_b200.build --checked`):
// device-side bounds / invariant checks that trap with the failing condition
// -- the stand-in for compute-sanitizer, which this GPU pool does not allow.
#ifdef DOPE_BOUNDS
#define DOPE_ASSERT(c)                                                                           \
    do {                                                                                         \
        if (!(c)) {                                                                              \
            printf("DOPE_ASSERT %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x, #c);                                                             \
            __trap();                                                                            \
        }                                                                                        \
    } while (0)
#else
#define DOPE_ASSERT(c) ((void)0)
#endif

namespace dope {

constexpr uint16_t HINF = 0xFFFF;

// storage of the integer path: y2 in {0,1,2} as bytes, multipliers as int16
typedef uint8_t ystore_t;
typedef int16_t astore_t;

// Programmatic dependent launch: wait for the preceding kernel in the stream
// (a no-op when this kernel was not launched with the PDL attribute), and
// let the next one launch once every CTA of this grid has called it.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ int byte_at(uint32_t w, int i) { return (int)((w >> (8 * i)) & 0xFFu); }
__device__ __forceinline__ void unpack_a4(uint2 v, int (&a)[4]) {
    a[0] = (int)(int16_t)(v.x & 0xFFFFu);
    a[1] = (int)(int16_t)(v.x >> 16);
    a[2] = (int)(int16_t)(v.y & 0xFFFFu);
    a[3] = (int)(int16_t)(v.y >> 16);
}
__device__ __forceinline__ uint2 pack_a4(int a0, int a1, int a2, int a3) {
    return make_uint2((uint32_t)(uint16_t)a0 | ((uint32_t)(uint16_t)a1 << 16),
                      (uint32_t)(uint16_t)a2 | ((uint32_t)(uint16_t)a3 << 16));
}
__device__ __forceinline__ uint32_t pack_y4(int y0, int y1, int y2, int y3) {
    return (uint32_t)y0 | ((uint32_t)y1 << 8) | ((uint32_t)y2 << 16) | ((uint32_t)y3 << 24);
}

// ---------------------------------------------------------------------------
// Geometry helpers (partition.py:62-77 with overlap 0)
// ---------------------------------------------------------------------------

struct Axis {
    int32_t dim, k, base, rem;
    __host__ __device__ void range(int32_t r, int32_t &lo, int32_t &len) const {
        lo = r * base + (r < rem ? r : rem);
        len = base + (r < rem ? 1 : 0);
    }
    __host__ __device__ int32_t owner(int32_t c) const {
        int32_t big = rem * (base + 1);
        return c < big ? c / (base + 1) : rem + (c - big) / base;
    }
};

__host__ __device__ inline Axis make_axis(int64_t dim, int32_t k) {
    Axis a;
    a.dim = (int32_t)dim;
    a.k = k;
    a.base = (int32_t)(dim / k);
    a.rem = (int32_t)(dim % k);
    return a;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// Bit-parallel BFS helpers (one warp).  The block's nodes are numbered
// v = r*BW + c over the padded box; bit v of the 64-bit word array is node v.
// Lane `l` owns words [l*WPL, (l+1)*WPL).
// ---------------------------------------------------------------------------

template <int WPL, int LANES, int T>
__device__ __forceinline__ uint64_t fetch_word(const uint64_t (&R)[WPL], int lane) {
    // word index lane*WPL + T  (T compile-time, may be negative)
    constexpr int DL = (T >= 0) ? (T / WPL) : -((-T + WPL - 1) / WPL);
    constexpr int SLOT = T - DL * WPL;
    uint64_t v = R[SLOT];
    if constexpr (DL > 0) {
        v = __shfl_down_sync(FULLMASK, v, DL);
        if (lane + DL >= LANES) v = 0;
    } else if constexpr (DL < 0) {
        v = __shfl_up_sync(FULLMASK, v, -DL);
        if (lane + DL < 0) v = 0;
    }
    return v;
}

// out[k] = bits of R shifted so that bit x holds R[x + S]  (S != 0)
template <int WPL, int LANES, int S, int K>
__device__ __forceinline__ uint64_t shifted(const uint64_t (&R)[WPL], int lane) {
    if constexpr (S > 0) {
        constexpr int Q = S / 64, REM = S % 64;
        uint64_t lo = fetch_word<WPL, LANES, K + Q>(R, lane);
        if constexpr (REM == 0) {
            return lo;
        } else {
            uint64_t hi = fetch_word<WPL, LANES, K + Q + 1>(R, lane);
            return (lo >> REM) | (hi << (64 - REM));
        }
    } else {
        constexpr int T = -S;
        constexpr int Q = T / 64, REM = T % 64;
        uint64_t hi = fetch_word<WPL, LANES, K - Q>(R, lane);
        if constexpr (REM == 0) {
            return hi;
        } else {
            uint64_t lo = fetch_word<WPL, LANES, K - Q - 1>(R, lane);
            return (hi << REM) | (lo >> (64 - REM));
        }
    }
}

// node v joins the reached set when it has a residual arc to an already
// reached node: direction d's mask holds "residual arc v -> v + off_d".
// Direction order: E(+1) W(-1) S(+BW) N(-BW) [D(+PL) U(-PL) in 3D].
template <int NW, int WPL, int LANES, int BW, int PL, bool DIAG, int K>
struct Expand {
    __device__ __forceinline__ static void run(const uint64_t (&R)[WPL], uint64_t (&NEW)[WPL],
                                               const uint64_t *__restrict__ m, int lane) {
        Expand<NW, WPL, LANES, BW, PL, DIAG, K - 1>::run(R, NEW, m, lane);
        const int idx = lane * WPL + (K - 1);
        const bool on = lane < LANES;
        uint64_t x = 0;
        const uint64_t e = on ? m[0 * NW + idx] : 0, w = on ? m[1 * NW + idx] : 0;
        const uint64_t sm = on ? m[2 * NW + idx] : 0, n = on ? m[3 * NW + idx] : 0;
        x = (e & shifted<WPL, LANES, 1, K - 1>(R, lane)) | (w & shifted<WPL, LANES, -1, K - 1>(R, lane)) |
            (sm & shifted<WPL, LANES, BW, K - 1>(R, lane)) | (n & shifted<WPL, LANES, -BW, K - 1>(R, lane));
        if constexpr (PL > 0) {
            const uint64_t dd = on ? m[4 * NW + idx] : 0, uu = on ? m[5 * NW + idx] : 0;
            x |= (dd & shifted<WPL, LANES, PL, K - 1>(R, lane)) | (uu & shifted<WPL, LANES, -PL, K - 1>(R, lane));
        }
        if constexpr (DIAG) {   // SE(+BW+1) NW(-BW-1) SW(+BW-1) NE(-BW+1)
            const uint64_t se = on ? m[4 * NW + idx] : 0, nw = on ? m[5 * NW + idx] : 0;
            const uint64_t sw = on ? m[6 * NW + idx] : 0, ne = on ? m[7 * NW + idx] : 0;
            x |= (se & shifted<WPL, LANES, BW + 1, K - 1>(R, lane)) |
                 (nw & shifted<WPL, LANES, -BW - 1, K - 1>(R, lane)) |
                 (sw & shifted<WPL, LANES, BW - 1, K - 1>(R, lane)) |
                 (ne & shifted<WPL, LANES, -BW + 1, K - 1>(R, lane));
        }
        NEW[K - 1] = x & ~R[K - 1];
    }
};
template <int NW, int WPL, int LANES, int BW, int PL, bool DIAG>
struct Expand<NW, WPL, LANES, BW, PL, DIAG, 0> {
    __device__ __forceinline__ static void run(const uint64_t (&)[WPL], uint64_t (&)[WPL],
                                               const uint64_t *__restrict__, int) {}
};

// Expand for 2D boxes whose rows are exactly one 64-bit word (BW == 64): the
// row above / below is the neighbouring word (one 64-bit shuffle per lane
// boundary), the diagonals are its 1-bit shifts -- about half the
// instructions of the generic shifted() form, which matters because one warp
// runs the BFS alone (its issue latency is the level time).
template <int NW, int WPL, bool DIAG>
__device__ __forceinline__ void expand_rows64(const uint64_t (&R)[WPL], uint64_t (&NEW)[WPL],
                                              const uint64_t *__restrict__ m, int lane) {
    static_assert(NW == 32 * WPL, "one lane owns WPL consecutive rows");
    uint64_t above = __shfl_up_sync(FULLMASK, R[WPL - 1], 1);
    uint64_t below = __shfl_down_sync(FULLMASK, R[0], 1);
    if (lane == 0) above = 0;
    if (lane == 31) below = 0;
#pragma unroll
    for (int k = 0; k < WPL; ++k) {
        const int idx = lane * WPL + k;
        const uint64_t own = R[k];
        const uint64_t up = k > 0 ? R[k - 1] : above;
        const uint64_t dn = k < WPL - 1 ? R[k + 1] : below;
        uint64_t x = (m[0 * NW + idx] & (own >> 1)) | (m[1 * NW + idx] & (own << 1)) |
                     (m[2 * NW + idx] & dn) | (m[3 * NW + idx] & up);
        if constexpr (DIAG)   // SE(+BW+1) NW(-BW-1) SW(+BW-1) NE(-BW+1)
            x |= (m[4 * NW + idx] & (dn >> 1)) | (m[5 * NW + idx] & (up << 1)) |
                 (m[6 * NW + idx] & (dn << 1)) | (m[7 * NW + idx] & (up >> 1));
        NEW[k] = x & ~own;
    }
}

// Global relabel: exact BFS distances to the sink set (g < 0) over residual
// arcs, written to h[] for nodes beyond the sink set (the caller has set
// h = 0 on the sink set and HINF elsewhere).  `masks` holds NDIR direction
// masks followed by the sink and active masks, NW words each.  Returns (on
// every lane of the calling warp) whether any active node (g > 0) is
// reached; `reach` receives the reached set.  Early exit once every active
// node has a level, except when there is none (then the BFS runs to
// completion and `reach` is the exact sink side).
template <int NW, int BW, int PL, bool DIAG = false>
__device__ int bfs_relabel(const uint64_t *__restrict__ masks, uint64_t *__restrict__ reach,
                           uint16_t *__restrict__ h, int lane, int *levels_out) {
    constexpr int NDIR = PL > 0 ? 6 : (DIAG ? 8 : 4);
    constexpr int LANES = NW < 32 ? NW : 32;
    constexpr int WPL = NW < 32 ? 1 : NW / 32;
    static_assert(NW % LANES == 0, "word layout");
    const uint64_t *mSink = masks + NDIR * NW, *mAct = masks + (NDIR + 1) * NW;
    const bool on = lane < LANES;
    uint64_t R[WPL], A[WPL], NEW[WPL];
    bool any_act = false;
#pragma unroll
    for (int k = 0; k < WPL; ++k) {
        const int idx = lane * WPL + k;
        R[k] = on ? mSink[idx] : 0;
        A[k] = on ? mAct[idx] : 0;
        any_act |= (A[k] != 0);
    }
    const bool have_active = __any_sync(FULLMASK, any_act);
    int level = 0;
    for (;;) {
        if (have_active) {
            bool missing = false;
#pragma unroll
            for (int k = 0; k < WPL; ++k) missing |= (A[k] & ~R[k]) != 0;
            if (!__any_sync(FULLMASK, missing)) break;
        }
        if constexpr (PL == 0 && BW == 64 && NW >= 32)
            expand_rows64<NW, WPL, DIAG>(R, NEW, masks, lane);
        else
            Expand<NW, WPL, LANES, BW, PL, DIAG, WPL>::run(R, NEW, masks, lane);
        bool grew = false;
#pragma unroll
        for (int k = 0; k < WPL; ++k) grew |= (NEW[k] != 0);
        if (!__any_sync(FULLMASK, grew)) break;
        ++level;
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            R[k] |= NEW[k];
            // heights only steer a following sweep: a BFS without active
            // nodes ends the solve (hit = false), its heights are never read
            uint64_t nb = have_active ? NEW[k] : 0ull;
            const int base = (lane * WPL + k) * 64;
            while (nb) {
                const int b = __ffsll((long long)nb) - 1;
                nb &= nb - 1;
                h[base + b] = (uint16_t)level;
            }
        }
    }
    bool hit = false;
#pragma unroll
    for (int k = 0; k < WPL; ++k) {
        if (on) reach[lane * WPL + k] = R[k];
        hit |= (A[k] & R[k]) != 0;
    }
    *levels_out = level;
    return __any_sync(FULLMASK, hit);
}

// Global relabel with bit-sliced levels: as bfs_relabel, but the level of a
// newly reached node is not stored per node by its owning lane (a serial loop
// over the frontier bits of a word: 8-connected wavefronts are squares whose
// top / bottom edges fill whole words) -- bit b of the level is OR-ed into
// plane b (planes[b * NW + word], zeroed by the caller) for the whole word at
// once.  levels_to_heights() then decodes the planes with every thread of the
// CTA.  Planes may alias the height array (decode stages through registers).
template <int NW, int BW, int PL, bool DIAG = false>
__device__ int bfs_relabel_planes(const uint64_t *__restrict__ masks, uint64_t *__restrict__ reach,
                                  uint64_t *__restrict__ planes, int lane, int *levels_out) {
    constexpr int NDIR = PL > 0 ? 6 : (DIAG ? 8 : 4);
    constexpr int LANES = NW < 32 ? NW : 32;
    constexpr int WPL = NW < 32 ? 1 : NW / 32;
    static_assert(NW % LANES == 0, "word layout");
    const uint64_t *mSink = masks + NDIR * NW, *mAct = masks + (NDIR + 1) * NW;
    const bool on = lane < LANES;
    uint64_t R[WPL], A[WPL], NEW[WPL];
    bool any_act = false;
#pragma unroll
    for (int k = 0; k < WPL; ++k) {
        const int idx = lane * WPL + k;
        R[k] = on ? mSink[idx] : 0;
        A[k] = on ? mAct[idx] : 0;
        any_act |= (A[k] != 0);
    }
    const bool have_active = __any_sync(FULLMASK, any_act);
    int level = 0;
    for (;;) {
        if (have_active) {
            bool missing = false;
#pragma unroll
            for (int k = 0; k < WPL; ++k) missing |= (A[k] & ~R[k]) != 0;
            if (!__any_sync(FULLMASK, missing)) break;
        }
        if constexpr (PL == 0 && BW == 64 && NW >= 32)
            expand_rows64<NW, WPL, DIAG>(R, NEW, masks, lane);
        else
            Expand<NW, WPL, LANES, BW, PL, DIAG, WPL>::run(R, NEW, masks, lane);
        bool grew = false;
#pragma unroll
        for (int k = 0; k < WPL; ++k) grew |= (NEW[k] != 0);
        if (!__any_sync(FULLMASK, grew)) break;
        ++level;
#pragma unroll
        for (int k = 0; k < WPL; ++k) R[k] |= NEW[k];
        if (have_active) {
            // heights only steer a following sweep (see bfs_relabel)
            for (int lv = level, b = 0; lv; lv >>= 1, ++b) {
                if (!(lv & 1)) continue;
#pragma unroll
                for (int k = 0; k < WPL; ++k)
                    if (on && NEW[k]) {
                        DOPE_ASSERT(b < 16 && (NEW[k] & R[k]) == NEW[k]);   // planes fit the height array
                        planes[b * NW + lane * WPL + k] |= NEW[k];
                    }
            }
        }
    }
    bool hit = false;
#pragma unroll
    for (int k = 0; k < WPL; ++k) {
        if (on) reach[lane * WPL + k] = R[k];
        hit |= (A[k] & R[k]) != 0;
    }
    *levels_out = level;
    return __any_sync(FULLMASK, hit);
}

// Every thread of the CTA: heights from the level planes of a BFS that ran
// `levels` levels (h = level for reached nodes -- 0 on the sink set -- HINF
// otherwise).  planes may alias h: the bits are gathered into registers,
// then -- behind a barrier -- the heights are written.
template <int M, int NT>
__device__ __forceinline__ void levels_to_heights(const uint64_t *planes, const uint64_t *__restrict__ reach,
                                                  uint16_t *h, int levels) {
    constexpr int NPT = M / NT, NW = M / 64;
    const int np = 32 - __clz(levels);
    DOPE_ASSERT(levels > 0 && levels < M && np <= 16);
    uint16_t hv[NPT];
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
        const int v = threadIdx.x + i * NT;
        const int word = v >> 6, bit = v & 63;
        uint32_t x = 0;
        for (int b = 0; b < np; ++b) x |= (uint32_t)((planes[b * NW + word] >> bit) & 1ull) << b;
        hv[i] = ((reach[word] >> bit) & 1ull) ? (uint16_t)x : HINF;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NPT; ++i) h[threadIdx.x + i * NT] = hv[i];
}

// ---------------------------------------------------------------------------
// Sharded mode: layout of a shard's halo buffer (dope_halo_bytes), U bytes per
// exchanged row (2D) / plane (3D): [0, U) first local row out, [U, 2U) last
// local row out, [2U, 3U) row received from above, [3U, 4U) from below, then
// (8-byte aligned) the int16 multipliers of the ghost row above and below,
// then (16-byte aligned) the peer-exchange flags: uint32 [row from above, row
// from below, K1 done-counter, pad, agg-slot flag of every shard].
// ---------------------------------------------------------------------------
__host__ __device__ inline int64_t halo_ga_offset(int64_t U) { return (4 * U + 7) / 8 * 8; }
__host__ __device__ inline int64_t halo_flag_offset(int64_t U) { return (halo_ga_offset(U) + 4 * U + 15) / 16 * 16; }
__host__ __device__ inline int64_t halo_bytes(int64_t U, int64_t count) {
    return halo_flag_offset(U) + 4 * (4 + (count > 0 ? count : 1));
}

// ---------------------------------------------------------------------------
// Per-iteration state digest (test / audit mode: dope_lattice.trace_hash).
// H_k = sum_g v_k(g) * mix64(3 (base + g) + k) mod 2^64 over the iteration's
// labels (k = 0), 2y (k = 1) and multipliers (k = 2): order-independent, so
// any reduction order -- and per-shard sums with a global index base -- give
// the words the CPU oracle computes (oracle/dope_oracle.c state_digest).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// One thread: open iteration st.iteration's digest slot unless it was already
// taken (a launch after the run stopped is a no-op).  h holds 3 * max_iters
// digest words followed by two control words: [last digested iteration, active].
template <typename State>
__global__ void k_digest_begin(const State *st, uint64_t *h, int max_iters) {
    const int it = st->iteration;
    uint64_t *ctl = h + 3 * (size_t)max_iters;
    if (it >= 1 && it <= max_iters && (int64_t)ctl[0] != it) {
        ctl[0] = (uint64_t)it;
        ctl[1] = 1;
        h[3 * (size_t)(it - 1)] = 0;
        h[3 * (size_t)(it - 1) + 1] = 0;
        h[3 * (size_t)(it - 1) + 2] = 0;
    } else {
        ctl[1] = 0;
    }
}

// y (k = 1) and a (k = 2) may be null (float path: only the labels are integers).
template <typename State, typename YT, typename AT>
__global__ void __launch_bounds__(256) k_digest(const State *st, uint64_t *h, int max_iters, int64_t n,
                                                int64_t base, const uint8_t *__restrict__ yhat,
                                                const YT *y0, const YT *y1, const YT *y2,
                                                const AT *__restrict__ a) {
    const uint64_t *ctl = h + 3 * (size_t)max_iters;
    if (!ctl[1]) return;
    const int64_t it = (int64_t)ctl[0];
    const int cur = st->ycur;
    const YT *__restrict__ y = cur == 0 ? y0 : (cur == 1 ? y1 : y2);
    uint64_t s0 = 0, s1 = 0, s2 = 0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t b = 3 * (uint64_t)(base + g);
        s0 += (uint64_t)yhat[g] * mix64(b);
        if (y) s1 += (uint64_t)(int64_t)y[g] * mix64(b + 1);
        if (a) s2 += (uint64_t)(int64_t)a[g] * mix64(b + 2);
    }
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_down_sync(FULLMASK, s0, o);
        s1 += __shfl_down_sync(FULLMASK, s1, o);
        s2 += __shfl_down_sync(FULLMASK, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *slot = reinterpret_cast<unsigned long long *>(h + 3 * (size_t)(it - 1));
        atomicAdd(slot, (unsigned long long)s0);
        atomicAdd(slot + 1, (unsigned long long)s1);
        atomicAdd(slot + 2, (unsigned long long)s2);
    }
}

}  // namespace dope
