// lattice3d_smem.cuh -- K1-3D with the whole 32^3 sub-region in shared memory.
// Included by dope_lattice.cu inside namespace dope, after lattice3d.cuh.
//
// The HBM-scratch kernel (lattice3d.cuh) pays an L2 round trip for every
// excess / height / residual access of every sweep.  Here a 32^3 block's
// residual graph is packed into 184 KB of shared memory:
//   * excess: int16, two per 32-bit word, biased by 2^15 so that a packed
//     atomicAdd of (delta << 16*half) never carries into the other half
//     (|excess| <= |2*linear| + 6*cap <= 32000 is checked per block; a block
//     that could leave the range runs the HBM-scratch body instead);
//   * heights: uint16;
//   * residuals of the E, S, D arcs only, 4 bits each (2*cap <= 15), eight per
//     word; the reverse arc's residual is 2cap - forward.  A push moves flow
//     on one edge, and only the higher endpoint of an edge can push in a
//     sweep, so a nibble has one writer per sweep; atomics only keep the
//     neighbouring nibbles of the same word intact;
//   * the global relabel runs on all 32 warps: warp w owns plane z = w, lane l
//     row y = l, one 32-bit reach word per row.  +-x is a shift, +-y a
//     shuffle, +-z a double-buffered shared row, one barrier per BFS level.
// Node-parallel phases (prologue, push, relabel, epilogue) map v = z*1024 +
// y*32 + x with z the loop index, y the warp and x the lane (conflict-free).
// Labels, flows and the exactness argument are those of DESIGN.md §2.

namespace k1s {
constexpr int B = 32, M = B * B * B, NT = 1024, PLANE = B * B;
constexpr int NIBW = M / 8;                                // nibble words per plane
constexpr size_t OFF_G = 0;                                // uint32[M/2] packed excess
constexpr size_t OFF_H = OFF_G + 2 * (size_t)M;            // uint16[M]
constexpr size_t OFF_F = OFF_H + 2 * (size_t)M;            // uint32[3][M/8] E,S,D residual nibbles
constexpr size_t OFF_R = OFF_F + 3 * 4 * (size_t)NIBW;     // uint32[2][1024] reach rows
constexpr size_t OFF_K = OFF_R + 2 * 4 * 1024;             // uint32[2][1024] sink / active rows
constexpr size_t OFF_SLOT = OFF_K + 2 * 4 * 1024;           // uint16[32 warps][32] batches
constexpr size_t OFF_FLAG = OFF_SLOT + 2 * 32 * 32;          // uint32[2][32] row-activity flags
constexpr size_t OFF_MISC = OFF_FLAG + 2 * 4 * 32;
constexpr size_t OFF_CAND = OFF_MISC + 64;                  // uint32[2][32 * 33] push / relabel candidate rows
constexpr int CPITCH = 33;                                  // word (y, z) = y * 33 + z: conflict-free by y and by z
constexpr size_t SMEM = OFF_CAND + 2 * 4 * 32 * CPITCH;
constexpr int UBR = M + 128;                               // int8 u brick: 128-byte header + box
constexpr int BIAS = 32768;
constexpr int GMAX = 32000;
static_assert(SMEM <= 227 * 1024, "shared memory");
static_assert(K1Cfg3<32, 32, 32, NT>::SMEM <= SMEM, "fallback body fits");
}  // namespace k1s

__device__ __forceinline__ int32_t s3_getg(const uint32_t *G2, int v) {
    return (int32_t)((G2[v >> 1] >> ((v & 1) << 4)) & 0xffffu) - k1s::BIAS;
}
__device__ __forceinline__ void s3_addg(uint32_t *G2, int v, int32_t d) {
    atomicAdd(&G2[v >> 1], (uint32_t)d << ((v & 1) << 4));
}
__device__ __forceinline__ int32_t s3_nib(const uint32_t *P, int v) {
    return (int32_t)((P[v >> 3] >> ((v & 7) << 2)) & 0xfu);
}
__device__ __forceinline__ void s3_addnib(uint32_t *P, int v, int32_t d) {
    atomicAdd(&P[v >> 3], (uint32_t)d << ((v & 7) << 2));
}
// eight nibbles -> eight bits (bit i set iff nibble i != 0)
__device__ __forceinline__ uint32_t s3_nz8(uint32_t x) {
    uint32_t t = (x | (x >> 1) | (x >> 2) | (x >> 3)) & 0x11111111u;
    t = (t | (t >> 3)) & 0x03030303u;
    t = (t | (t >> 6)) & 0x000F000Fu;
    return (t | (t >> 12)) & 0xFFu;
}
__device__ __forceinline__ uint32_t s3_nz32(uint4 w) {
    return s3_nz8(w.x) | (s3_nz8(w.y) << 8) | (s3_nz8(w.z) << 16) | (s3_nz8(w.w) << 24);
}
__device__ __forceinline__ uint4 s3_xor(uint4 w, uint32_t c) {
    return make_uint4(w.x ^ c, w.y ^ c, w.z ^ c, w.w ^ c);
}

__device__ __forceinline__ int64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}


__device__ __forceinline__ uint32_t s3_lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-level stream compaction: the set bits of `word` (lane i <-> node v of
// lane i) join the warp's batch `slots[0..cnt)`; every full batch of 32 runs
// `work(node)` with one node per lane.  Returns the new batch fill.
template <class F>
__device__ __forceinline__ int s3_enqueue(uint16_t *slots, uint32_t word, int cnt, int lane, int v, F &&work) {
    while (word) {
        const bool mine = (word >> lane) & 1u;
        const int rank = __popc(word & s3_lanemask_lt());
        const int room = 32 - cnt;
        if (mine && rank < room) slots[cnt + rank] = (uint16_t)v;
        const int n = __popc(word);
        word = __ballot_sync(FULLMASK, mine && rank >= room);
        if (n >= room) {
            __syncwarp();
            work((int)slots[lane]);
            __syncwarp();
            cnt = 0;
        } else {
            cnt += n;
        }
    }
    return cnt;
}

// candidate bitmasks of the sweeps: word (y, z) = y * CPITCH + z holds one bit per
// x, so warp y reads the words of its 32 rows with one load (lane = z) and the
// BFS owners (warp z, lane y) store theirs without bank conflicts
__device__ __forceinline__ void s3_mark(uint32_t *C, int v) {
    atomicOr(&C[((v >> 5) & 31) * k1s::CPITCH + (v >> 10)], 1u << (v & 31));
}

// push the excess of active node v along its admissible arcs (h[w] = h[v]-1),
// E W S N D U order; nodes that received excess or kept some become relabel
// candidates (Cr)
__device__ __forceinline__ void s3_push(uint32_t *G2, const uint16_t *h, uint32_t *FE, uint32_t *FS,
                                        uint32_t *FD, uint32_t *Cr, int v, int32_t cap2) {
    using namespace k1s;
    const int32_t e = s3_getg(G2, v);
    const uint16_t hv = h[v];
    if (e <= 0 || hv == HINF || hv == 0) return;
    const uint16_t ht = hv - 1;
    const int x = v & (B - 1), y = (v >> 5) & (B - 1), z = v >> 10;
    int32_t left = e;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        int32_t r;
        int w;
        if (d == 0) { r = s3_nib(FE, v); w = v + 1; }
        else if (d == 1) { if (x == 0) continue; r = cap2 - s3_nib(FE, v - 1); w = v - 1; }
        else if (d == 2) { r = s3_nib(FS, v); w = v + B; }
        else if (d == 3) { if (y == 0) continue; r = cap2 - s3_nib(FS, v - B); w = v - B; }
        else if (d == 4) { r = s3_nib(FD, v); w = v + PLANE; }
        else { if (z == 0) continue; r = cap2 - s3_nib(FD, v - PLANE); w = v - PLANE; }
        if (r == 0) continue;
        if (h[w] != ht) continue;
        const int32_t delta = left < r ? left : r;
        if (d == 0) s3_addnib(FE, v, -delta);
        else if (d == 1) s3_addnib(FE, w, delta);
        else if (d == 2) s3_addnib(FS, v, -delta);
        else if (d == 3) s3_addnib(FS, w, delta);
        else if (d == 4) s3_addnib(FD, v, -delta);
        else s3_addnib(FD, w, delta);
        s3_addg(G2, w, delta);
        s3_mark(Cr, w);
        left -= delta;
        if (left == 0) break;
    }
    if (left != e) s3_addg(G2, v, -(e - left));
    if (left) s3_mark(Cr, v);
}

// h[v] = 1 + min height over v's residual arcs (HINF when none or >= M);
// returns whether v stays below HINF
__device__ __forceinline__ int s3_relabel(const uint32_t *G2, uint16_t *h, const uint32_t *FE, const uint32_t *FS,
                                          const uint32_t *FD, uint32_t *Cp, int v, int32_t cap2) {
    using namespace k1s;
    if (s3_getg(G2, v) <= 0 || h[v] == HINF) return 0;   // a candidate without excess (a sink absorbed it)
    const int x = v & (B - 1), y = (v >> 5) & (B - 1), z = v >> 10;
    uint32_t mn = HINF;
    if (s3_nib(FE, v)) mn = min(mn, (uint32_t)h[v + 1]);
    if (x > 0 && s3_nib(FE, v - 1) != cap2) mn = min(mn, (uint32_t)h[v - 1]);
    if (s3_nib(FS, v)) mn = min(mn, (uint32_t)h[v + B]);
    if (y > 0 && s3_nib(FS, v - B) != cap2) mn = min(mn, (uint32_t)h[v - B]);
    if (s3_nib(FD, v)) mn = min(mn, (uint32_t)h[v + PLANE]);
    if (z > 0 && s3_nib(FD, v - PLANE) != cap2) mn = min(mn, (uint32_t)h[v - PLANE]);
    const uint32_t nh = (mn + 1 >= (uint32_t)M) ? HINF : mn + 1;
    if (nh != h[v]) h[v] = (uint16_t)nh;
    if (nh != HINF) s3_mark(Cp, v);   // pushes in the next sweep
    return nh != HINF;
}

// int8 copy of u in box order, one brick per sub-region after the fallback
// scratch (L.scratch + K*6M, stride UBR): the shared-memory K1 bulk-copies it
// in one piece instead of gathering 32-byte rows of int32.  Header byte 0 != 0:
// some |u| of the block exceeds int8 (that block runs the HBM-scratch body).
__device__ __forceinline__ int8_t *u_brick(const Lat2 &L, int k) {
    return reinterpret_cast<int8_t *>(L.scratch + (size_t)L.K * 6 * k1s::M + (size_t)k * k1s::UBR);
}

// out of line so that its registers do not count against the fast path
__device__ __noinline__ void mincut3d_l2_fallback(const Lat2 &L, const K1Tune &T, int k, uint8_t *smem) {
    mincut3d_l2<k1s::B, k1s::B, k1s::B, k1s::NT>(L, T, k, smem);
}

__global__ void __launch_bounds__(k1s::NT, 1) k_block_mincut3d_s(Lat2 L, K1Tune T) {
    using namespace k1s;
    extern __shared__ __align__(16) uint8_t sm3[];
    uint32_t *G2 = reinterpret_cast<uint32_t *>(sm3 + OFF_G);
    uint16_t *h = reinterpret_cast<uint16_t *>(sm3 + OFF_H);
    uint32_t *FE = reinterpret_cast<uint32_t *>(sm3 + OFF_F);
    uint32_t *FS = FE + NIBW, *FD = FE + 2 * NIBW;
    uint32_t *Rb = reinterpret_cast<uint32_t *>(sm3 + OFF_R);
    uint32_t *Kb = reinterpret_cast<uint32_t *>(sm3 + OFF_K);   // [0] sink rows, [1] active rows
    int *misc = reinterpret_cast<int *>(sm3 + OFF_MISC);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint16_t *slots = reinterpret_cast<uint16_t *>(sm3 + OFF_SLOT) + warp * 32;
    // row-activity flags: word y, bit z <=> row (z, y) may hold a node to push
    // (Fp) / to relabel (Fr); warp w scans the rows of word w
    uint32_t *Cp = reinterpret_cast<uint32_t *>(sm3 + OFF_CAND), *Cr = Cp + 32 * CPITCH;
    int k = blockIdx.x;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm3 + OFF_MISC + 32);
    if (L.dlist) {   // run loop: CTA i takes entry i of this iteration's dirty-block list
        const int stop = L.st->stop, it = L.st->iteration;
        const uint32_t *lst = dirty_list(L, it);
        if (blockIdx.x == 0 && tid == 0) dirty_list(L, it + 1)[0] = 0u;   // the next pass fills it
        const uint32_t cnt = lst[0], ent = lst[1 + blockIdx.x];
        if (stop || blockIdx.x >= cnt) {
            if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
            return;
        }
        k = (int)ent;
    } else if (L.st->stop || (L.skip_clean && L.dirty[k] == 0)) {
        if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
        return;
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        L.dirty[k] = 0;
        L.dirty[L.K + k] = (uint32_t)L.st->iteration + 1u;   // solve epoch (clean-block K2 pass)
    }
    // diagnostics (L.timeline): [0] start [1] end [2] rounds [3] sweeps
    // [4] prologue end [5] first relabel end [6] its levels [7] ns in relabels
    const bool tl = L.timeline && tid == 0;
    int64_t t_bfs = 0;
    if (tl) {
        const int64_t t = gtimer();
        L.timeline[8 * k + 0] = t;
        L.timeline[8 * k + 4] = t;
        L.timeline[8 * k + 5] = t;
    }

    int bz, by, bx;
    const Geo3 gb = block_geo3(L, k, bz, by, bx);
    const int32_t W = L.W, H = L.ay.dim, D = L.az.dim;
    const int64_t HW = (int64_t)H * W;
    const int32_t cap = L.cap, cap2 = 2 * cap;
    const astore_t *__restrict__ a_cur = L.a;
    const ystore_t *__restrict__ y_cur = L.y2[L.st->ycur];
    // persistent residuals: nibble planes E, S, D (uint32[3][M/8]) at the
    // start of the block's resid slot; the fallback body uses byte planes
    uint8_t *rr = L.resid + (size_t)k * 6 * M;
    uint32_t *gF = reinterpret_cast<uint32_t *>(rr);
    const bool up_z = gb.lo_z > 0 || L.gzu, dn_z = gb.lo_z + gb.dz < D || L.gzd;   // ghost planes: shards
    const bool up_r = gb.lo_r > 0, dn_r = gb.lo_r + gb.hr < H;
    const bool lf_c = gb.lo_c > 0, rt_c = gb.lo_c + gb.wc < W;
    const bool xin = lane < gb.wc, yin = warp < gb.hr;

    // ---- prologue ----
    // (1) the persistent E/S/D nibble planes (48 KB) stream in by one bulk copy
    //     while (2) 2*linear is computed from u, a, y; (3) then the excess adds
    //     the stored flow: excess = 2*linear + sum over the 6 arcs of (r - cap).
    const bool quads = L.q3 && (gb.lo_c % 4 == 0) && (gb.wc % 4 == 0);
    // the int8 u brick (quad path) lands in the height array, unused until the
    // first relabel
    const int8_t *ubs = reinterpret_cast<const int8_t *>(sm3 + OFF_H);
    if ((L.warm || quads) && tid == 0) {
        mbar_expect_tx(bar, (L.warm ? 3 * NIBW * 4 : 0) + (quads ? UBR : 0));
        if (L.warm) {
#pragma unroll
            for (int p = 0; p < 3; ++p)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                    ::"r"(smem_u32(FE + p * NIBW)), "l"(gF + p * NIBW), "r"(NIBW * 4), "r"(smem_u32(bar))
                    : "memory");
        }
        if (quads)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                ::"r"(smem_u32(ubs)), "l"(u_brick(L, k)), "r"(UBR), "r"(smem_u32(bar))
                : "memory");
    }
    int over = 0;
    const int32_t lim = GMAX - 6 * cap;
    if (quads) {
        // thread -> 4 consecutive x of one row; 128 rows per pass, 8 passes.
        const int x0 = (tid & 7) * 4;
        // u comes from the int8 brick; a, y of a pass (4 planes: 12 KB)
        // stream into a double-buffered staging area in the (not yet used)
        // height array by per-thread cp.async, two passes ahead; the cross-block neighbour words of the
        // next pass are register loads one pass ahead.  No register holds
        // in-flight data.  The stored flow's net inflow is added in the same
        // pass (the nibble planes arrive with pass 0).
        uint2 *stA = reinterpret_cast<uint2 *>(sm3 + OFF_H + UBR);   // [2][1024]
        uint32_t *stY = reinterpret_cast<uint32_t *>(stA + 2 * NT);  // [2][1024]
        static_assert(UBR + 2 * NT * 12 <= 2 * M, "u brick + staging fit the height array");
        auto gidx = [&](int p, bool &ok, int &z, int &y) -> int64_t {
            const int row = p * 128 + (tid >> 3);
            z = row >> 5;
            y = row & 31;
            ok = z < gb.dz && y < gb.hr && x0 < gb.wc;
            return ((int64_t)(gb.lo_z + z) * H + gb.lo_r + y) * W + gb.lo_c + x0;
        };
        auto issue = [&](int p) {
            bool ok;
            int z, y;
            const int64_t G = gidx(p, ok, z, y);
            const int b = p & 1;
            if (ok) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(stA + b * NT + tid)),
                             "l"(a_cur + G) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(stY + b * NT + tid)),
                             "l"(y_cur + G) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // cross-block neighbour words of pass p (one row per axis; the
        // 1-thick-block second side is read in the compute step)
        auto nbr = [&](int p, uint32_t &ny, uint32_t &nz, uint32_t &nx) {
            bool ok;
            int z, y;
            const int64_t G = gidx(p, ok, z, y);
            ny = nz = nx = 0;
            if (!ok) return;
            if (y == 0 && up_r) ny = *reinterpret_cast<const uint32_t *>(y_cur + G - W);
            else if (y == gb.hr - 1 && dn_r) ny = *reinterpret_cast<const uint32_t *>(y_cur + G + W);
            if (z == 0 && up_z) nz = *reinterpret_cast<const uint32_t *>(y_cur + G - HW);
            else if (z == gb.dz - 1 && dn_z) nz = *reinterpret_cast<const uint32_t *>(y_cur + G + HW);
            if (x0 == 0 && lf_c) nx = y_cur[G - 1];
            if (x0 + 4 == gb.wc && rt_c) nx |= (uint32_t)y_cur[G + 4] << 8;
        };
        issue(0);
        issue(1);
        uint32_t ny, nz, nx;
        nbr(0, ny, nz, nx);
        mbar_wait(bar, 0);   // u brick (+ the nibble planes: flow terms are added in the same passes)
#ifdef K1S_DIAG
        if (tl) L.timeline[8 * k + 7] = gtimer();
#endif
        if (ubs[0]) over = 1;  // some |u| exceeds int8: the HBM-scratch body solves this block
        // fully unrolled: a register move of a pending load result would
        // wait for it, exposing one DRAM latency per pass
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
            uint32_t ny1 = 0, nz1 = 0, nx1 = 0;
            if (pp + 1 < 8) nbr(pp + 1, ny1, nz1, nx1);   // in flight during this pass
            if (pp + 1 < 8) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            const int row = pp * 128 + (tid >> 3), z = row >> 5, y = row & 31;
            const int bsel = pp & 1;
            uint32_t uw = 0;
            uint2 a4 = make_uint2(0, 0);
            uint32_t y4 = 0;
            if (z < gb.dz && y < gb.hr && x0 < gb.wc) {
                uw = *reinterpret_cast<const uint32_t *>(ubs + 128 + z * PLANE + y * B + x0);
                a4 = stA[bsel * NT + tid];
                y4 = stY[bsel * NT + tid];
            }
            {
                const int v0 = z * PLANE + y * B + x0;
                const bool valid = z < gb.dz && y < gb.hr && x0 < gb.wc;
                int32_t g[4] = {0, 0, 0, 0};
                if (valid) {
                    const bool yb = (y == 0 && up_r), yt = (y == gb.hr - 1 && dn_r);
                    const bool zb = (z == 0 && up_z), zt = (z == gb.dz - 1 && dn_z);
                    int32_t yv[4], sx[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        yv[e] = (int32_t)((y4 >> (8 * e)) & 0xffu);
                        const int32_t by = (int32_t)((ny >> (8 * e)) & 0xffu);
                        const int32_t bz = (int32_t)((nz >> (8 * e)) & 0xffu);
                        sx[e] = ((yb || yt) ? yv[e] - by : 0) + ((zb || zt) ? yv[e] - bz : 0);
                    }
                    if (yb && yt) {   // 1-row block with neighbours on both sides
                        const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + y) * W + gb.lo_c + x0;
                        const uint32_t o = *reinterpret_cast<const uint32_t *>(y_cur + G + W);
#pragma unroll
                        for (int e = 0; e < 4; ++e) sx[e] += yv[e] - (int32_t)((o >> (8 * e)) & 0xffu);
                    }
                    if (zb && zt) {
                        const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + y) * W + gb.lo_c + x0;
                        const uint32_t o = *reinterpret_cast<const uint32_t *>(y_cur + G + HW);
#pragma unroll
                        for (int e = 0; e < 4; ++e) sx[e] += yv[e] - (int32_t)((o >> (8 * e)) & 0xffu);
                    }
                    if (x0 == 0 && lf_c) sx[0] += yv[0] - (int32_t)(nx & 0xffu);
                    if (x0 + 4 == gb.wc && rt_c) sx[3] += yv[3] - (int32_t)((nx >> 8) & 0xffu);
                    const int32_t uu[4] = {(int32_t)(int8_t)(uw & 0xffu), (int32_t)(int8_t)((uw >> 8) & 0xffu),
                                           (int32_t)(int8_t)((uw >> 16) & 0xffu), (int32_t)(int8_t)(uw >> 24)};
                    const uint32_t aw[2] = {a4.x, a4.y};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int32_t av = (int32_t)(int16_t)((aw[e >> 1] >> (16 * (e & 1))) & 0xffffu);
                        g[e] = 2 * uu[e] + L.lamw * sx[e] + L.mu * (2 * av - yv[e]) + L.mu;
                        over |= (g[e] > lim) | (g[e] < -lim);
                    }
                    if (L.warm) {
                        // excess += sum over the node's arcs of (r - cap), four
                        // nodes at once on bytes: per direction the forward
                        // arc's r minus the backward arc's (= 2cap - r of the
                        // neighbour's forward arc, the caps cancel).  A missing
                        // backward arc reads as cap, a missing forward arc
                        // (stored 0) gets cap added back: both terms vanish.
                        const int xs = (x0 & 7) * 4;   // bit offset of the quad in its nibble word
                        const int wi = v0 >> 3;
                        const uint32_t cw = (uint32_t)cap * 0x1111u;
                        const uint32_t wEc = FE[wi];
                        const uint32_t E4 = (wEc >> xs) & 0xFFFFu;
                        const uint32_t pn = x0 == 0 ? (uint32_t)cap
                                                    : (xs ? (wEc >> (xs - 4)) & 0xFu : FE[wi - 1] >> 28);
                        const uint32_t Ep4 = ((E4 << 4) | pn) & 0xFFFFu;
                        const uint32_t S4 = (FS[wi] >> xs) & 0xFFFFu;
                        const uint32_t N4 = y > 0 ? (FS[wi - B / 8] >> xs) & 0xFFFFu : cw;
                        const uint32_t D4 = (FD[wi] >> xs) & 0xFFFFu;
                        const uint32_t U4 = z > 0 ? (FD[wi - PLANE / 8] >> xs) & 0xFFFFu : cw;
                        uint32_t corr = x0 + 4 == gb.wc ? (uint32_t)cap << 24 : 0u;
                        if (y + 1 == gb.hr) corr += (uint32_t)cap * 0x01010101u;
                        if (z + 1 == gb.dz) corr += (uint32_t)cap * 0x01010101u;
                        auto spread4 = [](uint32_t x) -> uint32_t {   // 4 nibbles -> 4 bytes
                            uint32_t t = (x | (x << 8)) & 0x00FF00FFu;
                            return (t | (t << 4)) & 0x0F0F0F0Fu;
                        };
                        // bytes: flow + 48 (no carry / borrow: 0 < . < 256)
                        const uint32_t t4 = (spread4(E4) + spread4(S4) + spread4(D4) + corr + 0x30303030u) -
                                            (spread4(Ep4) + spread4(N4) + spread4(U4));
#pragma unroll
                        for (int e = 0; e < 4; ++e) g[e] += (int32_t)((t4 >> (8 * e)) & 0xffu) - 48;
                    }
                }
                if (!L.warm) {   // cold residual graph: every existing arc at cap
                    uint32_t nE = 0, nS = 0, nD = 0;
                    if (valid) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if (x0 + e + 1 < gb.wc) nE |= (uint32_t)cap << (4 * e);
                            if (y + 1 < gb.hr) nS |= (uint32_t)cap << (4 * e);
                            if (z + 1 < gb.dz) nD |= (uint32_t)cap << (4 * e);
                        }
                    }
                    reinterpret_cast<uint16_t *>(FE)[v0 >> 2] = (uint16_t)nE;
                    reinterpret_cast<uint16_t *>(FS)[v0 >> 2] = (uint16_t)nS;
                    reinterpret_cast<uint16_t *>(FD)[v0 >> 2] = (uint16_t)nD;
                }
                uint2 gw;
                gw.x = ((uint32_t)(g[0] + BIAS) & 0xffffu) | ((uint32_t)(g[1] + BIAS) << 16);
                gw.y = ((uint32_t)(g[2] + BIAS) & 0xffffu) | ((uint32_t)(g[3] + BIAS) << 16);
                *reinterpret_cast<uint2 *>(G2 + (v0 >> 1)) = gw;
            }
            if (pp + 2 < 8) issue(pp + 2);   // this thread's own slots: no barrier
            ny = ny1;
            nz = nz1;
            nx = nx1;
        }
#ifdef K1S_DIAG
        if (tl) L.timeline[8 * k + 6] = gtimer();
#endif
    } else {
        // scalar prologue (blocks whose x range is not quad-aligned): lane = x
#pragma unroll 2
        for (int z = 0; z < B; ++z) {
            const int v = z * PLANE + tid;
            const bool valid = xin && yin && z < gb.dz;
            int32_t gv = 0;
            if (valid) {
                const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + warp) * W + gb.lo_c + lane;
                const int32_t yg = (int32_t)y_cur[G];
                int32_t sx = 0;
                if (lane == 0 && lf_c) sx += yg - y_cur[G - 1];
                if (lane == gb.wc - 1 && rt_c) sx += yg - y_cur[G + 1];
                if (warp == 0 && up_r) sx += yg - y_cur[G - W];
                if (warp == gb.hr - 1 && dn_r) sx += yg - y_cur[G + W];
                if (z == 0 && up_z) sx += yg - y_cur[G - HW];
                if (z == gb.dz - 1 && dn_z) sx += yg - y_cur[G + HW];
                gv = 2 * L.u[G] + L.lamw * sx + L.mu * (2 * (int32_t)a_cur[G] - yg) + L.mu;
                over |= (gv > lim) | (gv < -lim);
            }
            if (!L.warm) {
                const uint32_t sh = (lane & 7) << 2;
                uint32_t nE = (valid && lane + 1 < gb.wc) ? (uint32_t)cap << sh : 0u;
                uint32_t nS = (valid && warp + 1 < gb.hr) ? (uint32_t)cap << sh : 0u;
                uint32_t nD = (valid && z + 1 < gb.dz) ? (uint32_t)cap << sh : 0u;
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    nE |= __shfl_xor_sync(FULLMASK, nE, o);
                    nS |= __shfl_xor_sync(FULLMASK, nS, o);
                    nD |= __shfl_xor_sync(FULLMASK, nD, o);
                }
                if ((lane & 7) == 0) {
                    FE[v >> 3] = nE;
                    FS[v >> 3] = nS;
                    FD[v >> 3] = nD;
                }
            }
            const uint32_t gb16 = (uint32_t)(gv + BIAS) & 0xffffu;
            const uint32_t hi = __shfl_down_sync(FULLMASK, gb16, 1);
            if ((lane & 1) == 0) G2[v >> 1] = gb16 | (hi << 16);
        }
        if (L.warm) {
            mbar_wait(bar, 0);
#pragma unroll 2
            for (int z = 0; z < B; ++z) {
                const int v = z * PLANE + tid;
                int32_t f = 0;
                if (xin && yin && z < gb.dz) {
                    if (lane + 1 < gb.wc) f += s3_nib(FE, v) - cap;
                    if (lane > 0) f += cap - s3_nib(FE, v - 1);
                    if (warp + 1 < gb.hr) f += s3_nib(FS, v) - cap;
                    if (warp > 0) f += cap - s3_nib(FS, v - B);
                    if (z + 1 < gb.dz) f += s3_nib(FD, v) - cap;
                    if (z > 0) f += cap - s3_nib(FD, v - PLANE);
                }
                const int32_t fo = __shfl_down_sync(FULLMASK, f, 1);
                if ((lane & 1) == 0) G2[v >> 1] += (uint32_t)f + ((uint32_t)fo << 16);
            }
        }
    }
    if (__syncthreads_or(over)) {
        // this block's excess could leave int16: solve it with the HBM-scratch
        // body on byte planes, then repack its E/S/D residuals as nibbles
        if (L.warm) {
            // forward planes from the nibbles; reverse planes zeroed (the body
            // derives the existing ones; the others must read as "no arc")
            for (int v = tid; v < M; v += NT) {
                rr[v] = (uint8_t)s3_nib(FE, v);
                rr[M + v] = 0;
                rr[2 * M + v] = (uint8_t)s3_nib(FS, v);
                rr[3 * M + v] = 0;
                rr[4 * M + v] = (uint8_t)s3_nib(FD, v);
                rr[5 * M + v] = 0;
            }
        }
        __syncthreads();
        mincut3d_l2_fallback(L, T, k, sm3);
        if (L.warm) {
            __syncthreads();
            for (int w = tid; w < 3 * NIBW; w += NT) {
                const int p = w / NIBW, v0 = (w - p * NIBW) * 8;
                uint32_t x = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e) x |= (uint32_t)rr[2 * p * M + v0 + e] << (4 * e);
                FE[w] = x;
            }
            __syncthreads();
            for (int w = tid; w < 3 * NIBW; w += NT) gF[w] = FE[w];
        }
        if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
        return;
    }

    if (tl) L.timeline[8 * k + 4] = gtimer();
    // row geometry of the BFS ownership (z = warp, y = lane)
    const int oz = warp, oy = lane;
    const bool rvalid = oz < gb.dz && oy < gb.hr;
    const uint32_t xmask = gb.wc >= 32 ? 0xffffffffu : ((1u << gb.wc) - 1u);
    const uint32_t existE = rvalid ? (xmask >> 1) : 0u;
    const uint32_t existS = (rvalid && oy + 1 < gb.hr) ? xmask : 0u;
    const uint32_t full = (uint32_t)cap2 * 0x11111111u;
    const int rowv = oz * PLANE + oy * B;   // first node of the owned row

    int rounds = 0;
    long long sweeps_done = 0;
    uint32_t R = 0;
    for (;;) {
        // ---- sink / active rows and initial heights (node-parallel) ----
        // eight nodes of a row per thread (one 16-byte load of packed excess, one
        // 16-byte store of heights; the four lanes of a row OR their mask bytes):
        // 4 passes instead of 32 ballot passes over the 32768 nodes.  Biased
        // halves: g < 0 <=> bit 15 clear; g > 0 <=> bit 15 set and low bits != 0.
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int item = i * NT + tid, rho = item >> 2, qd = item & 3;
            const int v0 = rho * B + 8 * qd;
            const uint4 w4 = *reinterpret_cast<const uint4 *>(G2 + (v0 >> 1));
            const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
            uint32_t hw[4], neg8 = 0, pos8 = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t w = ws[j];
                const uint32_t sg = w & 0x80008000u;             // sign bits: g >= 0
                hw[j] = (sg >> 15) * 0xFFFFu;                    // g < 0 -> 0, else HINF
                const uint32_t ng = ~w & 0x80008000u;
                neg8 |= (((ng >> 15) & 1u) | ((ng >> 30) & 2u)) << (2 * j);
                const uint32_t p0 = ((w >> 15) & 1u) & ((w & 0x7fffu) != 0u ? 1u : 0u);
                const uint32_t p1 = (w >> 31) & ((w & 0x7fff0000u) != 0u ? 1u : 0u);
                pos8 |= (p0 | (p1 << 1)) << (2 * j);
            }
            *reinterpret_cast<uint4 *>(h + v0) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            uint32_t bK = neg8 << (8 * qd), bA = pos8 << (8 * qd);
            bK |= __shfl_xor_sync(FULLMASK, bK, 1);
            bA |= __shfl_xor_sync(FULLMASK, bA, 1);
            bK |= __shfl_xor_sync(FULLMASK, bK, 2);
            bA |= __shfl_xor_sync(FULLMASK, bA, 2);
            if (qd == 0) {
                Kb[rho] = bK;            // rho = z * B + y
                Kb[1024 + rho] = bA;
            }
        }
        if (tid == 0) { misc[0] = 0; misc[1] = 0; misc[2] = 0; }
        __syncthreads();
        // ---- direction masks of the owned row from the nibble planes ----
        const uint4 wE = *reinterpret_cast<const uint4 *>(FE + (rowv >> 3));
        const uint4 wS = *reinterpret_cast<const uint4 *>(FS + (rowv >> 3));
        const uint4 wD = *reinterpret_cast<const uint4 *>(FD + (rowv >> 3));
        const uint32_t mE = s3_nz32(wE);
        const uint32_t mW = (s3_nz32(s3_xor(wE, full)) & existE) << 1;
        const uint32_t mS = s3_nz32(wS);
        const uint32_t mD = s3_nz32(wD);
        const uint32_t nfS = s3_nz32(s3_xor(wS, full)) & existS;   // arc (y+1) -> y has residual
        uint32_t mN = __shfl_up_sync(FULLMASK, nfS, 1);
        if (oy == 0) mN = 0;
        uint32_t mU = 0;
        if (oz > 0) {
            const uint4 wU = *reinterpret_cast<const uint4 *>(FD + ((rowv - PLANE) >> 3));
            const uint32_t exU = (rvalid && oz - 1 < gb.dz) ? xmask : 0u;
            mU = s3_nz32(s3_xor(wU, full)) & exU;
        }
        const int64_t t0 = tl ? gtimer() : 0;
        R = Kb[oz * B + oy];
        const uint32_t A = Kb[1024 + oz * B + oy];
        const bool have_active = __syncthreads_or(A != 0);
        Rb[oz * B + oy] = R;
        __syncthreads();

        // ---- global relabel: BFS over residual arcs from the sink set ----
        int level = 0, cur = 0;
        for (;;) {
            const uint32_t *Rc = Rb + cur * 1024;
            const uint32_t ryp = __shfl_down_sync(FULLMASK, R, 1), rym = __shfl_up_sync(FULLMASK, R, 1);
            const uint32_t rzp = oz + 1 < B ? Rc[(oz + 1) * B + oy] : 0u;
            const uint32_t rzm = oz > 0 ? Rc[(oz - 1) * B + oy] : 0u;
            const uint32_t nw = ((mE & (R >> 1)) | (mW & (R << 1)) | (mS & ryp) | (mN & rym) | (mD & rzp) |
                                 (mU & rzm)) & ~R;
            R |= nw;
            Rb[(cur ^ 1) * 1024 + oz * B + oy] = R;
            const int lv = level + 1;
            uint32_t b = nw;
            while (b) {
                const int x = __ffs(b) - 1;
                b &= b - 1;
                h[rowv + x] = (uint16_t)lv;
            }
            const uint32_t fl = (nw != 0 ? 1u : 0u) | ((A & ~R) != 0 ? 2u : 0u);
            const uint32_t wf = __reduce_or_sync(FULLMASK, fl);
            const int slot = level % 3;
            if (lane == 0 && wf) atomicOr(reinterpret_cast<unsigned *>(&misc[slot]), wf);
            if (tid == 0) misc[(level + 1) % 3] = 0;
            __syncthreads();
            const int f = misc[slot];
            if (f & 1) level = lv;
            cur ^= 1;
            if (!(f & 1)) break;                  // no growth: BFS complete
            if (have_active && !(f & 2)) break;   // every active node has a height
        }
        // sweep candidates: C (push from) = the active nodes the BFS reached, N (relabel) empty
        Cp[oy * CPITCH + oz] = A & R;
        Cr[oy * CPITCH + oz] = 0u;
        const int hit = __syncthreads_or((A & R) != 0);
        if (tl) {
            const int64_t t1 = gtimer();
            t_bfs += t1 - t0;
            if (rounds == 0) {
                L.timeline[8 * k + 5] = t1;
#ifndef K1S_DIAG
                L.timeline[8 * k + 6] = level;
#endif
            }
        }
        if (!hit) break;
        if (++rounds > T.max_rounds) {
            if (tid == 0) atomicCAS(&L.st->error, 0, k + 1);
            break;
        }
        // ---- push / relabel sweeps ----
        const int cap_sweeps = T.sweep_min + T.sweep_mul * level;
        for (int sw = 0; sw < cap_sweeps; ++sw) {
            ++sweeps_done;
            // push from C, then relabel N: warp y reads the candidate words of
            // its 32 rows (lane = z) in one load and packs the set bits into
            // batches of 32, one node per lane (no per-row scan of h and g)
            int cnt = 0;
            uint32_t cw = Cp[warp * CPITCH + lane];
            if (cw) Cp[warp * CPITCH + lane] = 0u;
            uint32_t rows = __ballot_sync(FULLMASK, cw != 0u);
            while (rows) {
                const int z = __ffs(rows) - 1;
                rows &= rows - 1;
                const uint32_t word = __shfl_sync(FULLMASK, cw, z);
                cnt = s3_enqueue(slots, word, cnt, lane, z * PLANE + tid,
                                 [&](int u) { s3_push(G2, h, FE, FS, FD, Cr, u, cap2); });
            }
            if (cnt) {
                __syncwarp();
                if (lane < cnt) s3_push(G2, h, FE, FS, FD, Cr, slots[lane], cap2);
                __syncwarp();
            }
            __syncthreads();
            int act = 0;
            cnt = 0;
            cw = Cr[warp * CPITCH + lane];
            if (cw) Cr[warp * CPITCH + lane] = 0u;
            rows = __ballot_sync(FULLMASK, cw != 0u);
            while (rows) {
                const int z = __ffs(rows) - 1;
                rows &= rows - 1;
                const uint32_t word = __shfl_sync(FULLMASK, cw, z);
                cnt = s3_enqueue(slots, word, cnt, lane, z * PLANE + tid,
                                 [&](int u) { act |= s3_relabel(G2, h, FE, FS, FD, Cp, u, cap2); });
            }
            if (cnt) {
                __syncwarp();
                if (lane < cnt) act |= s3_relabel(G2, h, FE, FS, FD, Cp, slots[lane], cap2);
                __syncwarp();
            }
            if (!__syncthreads_or(act)) break;
        }
    }
    // ---- epilogue: labels (sink side) and the E/S/D residual planes ----
    Rb[oz * B + oy] = R;
    __syncthreads();
    if (quads && (W & 3) == 0) {
        // four labels per 32-bit store: thread -> 4 consecutive x of one row,
        // 128 rows per pass (the quad prologue's mapping)
        const int x0 = (tid & 7) * 4;
#pragma unroll 4
        for (int p = 0; p < 8; ++p) {
            const int row = p * 128 + (tid >> 3), z = row >> 5, y = row & 31;
            if (!(z < gb.dz && y < gb.hr && x0 < gb.wc)) continue;
            const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + y) * W + gb.lo_c + x0;
            const uint32_t b = (Rb[z * B + y] >> x0) & 0xFu;
            *reinterpret_cast<uint32_t *>(L.yhat + G) = (b * 0x00204081u) & 0x01010101u;
        }
    } else {
#pragma unroll 4
        for (int z = 0; z < B; ++z) {
            if (!(xin && yin && z < gb.dz)) continue;
            const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + warp) * W + gb.lo_c + lane;
            L.yhat[G] = (uint8_t)((Rb[z * B + warp] >> lane) & 1u);
        }
    }
    if (L.warm && sweeps_done > 0) {   // E/S/D nibble planes back (48 KB; unchanged without a sweep)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int w = (j * NT + tid) * 4;
            *reinterpret_cast<uint4 *>(gF + w) = *reinterpret_cast<const uint4 *>(FE + w);
        }
    }
    if (tl) {
        L.timeline[8 * k + 1] = gtimer();
        L.timeline[8 * k + 2] = rounds;
        L.timeline[8 * k + 3] = sweeps_done;
#ifndef K1S_DIAG
        L.timeline[8 * k + 7] = t_bfs;
#endif
    }
    if (tid == 0) {
        atomicAdd((unsigned long long *)&L.st->solves, 1ull);
        atomicAdd((unsigned long long *)&L.st->sweeps, (unsigned long long)sweeps_done);
        atomicMax(&L.st->max_rounds_seen, rounds);
    }
    if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
}

// cold residual graph in the nibble layout: every existing E/S/D arc at cap
// fills the u bricks (dope_admm_init)
__global__ void k_init_ubrick(Lat2 L) {
    using namespace k1s;
    const int k = blockIdx.x;
    int bz, by, bx;
    const Geo3 gb = block_geo3(L, k, bz, by, bx);
    int8_t *ub = u_brick(L, k);
    const int64_t HW = (int64_t)L.ay.dim * L.W;
    int bad = 0;
    for (int v = threadIdx.x; v < M; v += blockDim.x) {
        const int z = v / PLANE, r = (v / B) % B, c = v % B;
        int32_t uv = 0;
        if (z < gb.dz && r < gb.hr && c < gb.wc)
            uv = L.u[(int64_t)(gb.lo_z + z) * HW + (int64_t)(gb.lo_r + r) * L.W + gb.lo_c + c];
        bad |= (uv < -128) | (uv > 127);
        ub[128 + v] = (int8_t)uv;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) ub[0] = (int8_t)(bad ? 1 : 0);
}

__global__ void k_init_resid3d_nib(Lat2 L) {
    using namespace k1s;
    const int k = blockIdx.x;
    int bz, by, bx;
    const Geo3 gb = block_geo3(L, k, bz, by, bx);
    uint32_t *gF = reinterpret_cast<uint32_t *>(L.resid + (size_t)k * 6 * M);
    for (int w = threadIdx.x; w < 3 * NIBW; w += blockDim.x) {
        const int p = w / NIBW, v0 = (w - p * NIBW) * 8;
        const int z = v0 / PLANE, r = (v0 / B) % B, c0 = v0 % B;
        // nibbles e with an existing arc: x = c0 + e inside the row (E: x + 1 inside)
        int n = 0;
        if (z < gb.dz && r < gb.hr) {
            if (p == 0) n = gb.wc - 1 - c0;
            else if ((p == 1 && r + 1 < gb.hr) || (p == 2 && z + 1 < gb.dz)) n = gb.wc - c0;
        }
        n = n < 0 ? 0 : (n > 8 ? 8 : n);
        const uint32_t m = n == 8 ? 0xffffffffu : ((1u << (4 * n)) - 1u);
        gF[w] = ((uint32_t)L.cap * 0x11111111u) & m;
    }
}
