// sweep_split.cu — the block-Thomas sweep for b = 16 (config 2's storage), third generation.
//
// Same recursion, twisted variant, SPIKE chunk slots and epilogue as sweep_small.cu:
//   forward : y_l = S_l^{-1} Y_l - H_l y_{l-1}
//   middle  : x_k = T^{-1} Y_k - (T^{-1}C_{k-1}) y_{k-1} [- (T^{-1}C_k^T) u_{k+1}]
//   backward: x_l = y_l - G_l x_{l+1}
//   epilogue: T = Re(c x) (real mode) or W = x (complex mode)
//
// The ncu capture of the 2-warp kernel (profiles/r02_cfg2_full.ncu-rep) showed what bounds a
// step of the dependent chain: one warp issues a DMMA every 16 clocks at best (the FP64 pipe of
// its SM sub-partition), and a step's 20 DMMAs per warp sat on the chain one after the other,
// with the other sub-partitions of the SM idle. So here
//   * each 8 x 8 output tile is computed by TWO warps, one for the real and one for the
//     imaginary part of the complex product: a 16-row block of 8 columns runs on 4 warps, one
//     per sub-partition, and a step's chain carries 8 (backward) or 8 + 4 (forward) DMMAs per
//     warp. The running vector is kept NEGATED and PLANAR in shared memory (u = -y; a real and
//     an imaginary plane), so both warps use the complex A fragment exactly as one 16-byte load
//     delivers it and differ only in which plane feeds which operand and in one sign at the fold:
//         re warp: P += a.re u.re, Q += a.im u.im, value = P - Q
//         im warp: P += a.re u.im, Q += a.im u.re, value = P + Q
//   * the step is software-pipelined: everything of step v + 1 that does not depend on the
//     running vector (waiting for its factor blocks, the S^{-1} Y product, loading the A
//     fragments of the dependent product) is issued behind step v's dependent DMMAs, before
//     step v's result is folded and stored, so only  barrier -> vector loads -> 8 DMMAs ->
//     fold -> store  remains on the chain;
//   * the producer warp streams factor blocks into a ring of single-block slots (a forward
//     step takes two, a backward step one) and the right-hand-side tile of a forward step as
//     one bulk copy per column, all completing on the step's mbarrier; the column blocks of a
//     node take turns prefetching the factor blocks into L2 far ahead of the ring
//     (cp.async.bulk.prefetch.L2), so a ring refill is an L2 hit; the backward's y_l comes
//     back through a lane-private cp.async ring (each lane re-reads the component it stored);
//   * the quadrature epilogue T = Re(c x) needs both components, so it runs one step late from
//     the shared running vector, one element per thread with coalesced column stores;
//   * all ring positions, parities and global pointers advance incrementally (no per-step
//     division or multiplication by runtime values).

#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "mbarrier.cuh"

namespace cg = cooperative_groups;

namespace feastgpu {

template <int B, int NC, bool CPLX_IN, bool TW>
struct SplitShape {
  static constexpr int MT = B / 8, NT = NC / 8, KQ = B / 4;
  static constexpr int NCW = MT * NT * 2;    // compute warps: (row tile, column tile, re | im)
  static constexpr int NTHR = (NCW + 1) * 32;
  static constexpr int NSLOT = 10;           // factor-block ring (even: a forward step takes 2)
  static constexpr int NRHS = NSLOT / 2;     // right-hand-side tiles, one per forward step in flight
  static constexpr int RY = 8;               // lane-private y ring (backward), RY - 1 steps ahead
  static constexpr int SV = B + 4;           // running vector plane [col][k] stride (double)
  static constexpr int RS = B + 4;           // right-hand-side tile [col][k] stride (elements)
  static constexpr int RELB = CPLX_IN ? 16 : 8;
  static constexpr int BB = B * B;
  static constexpr int PLANE = NC * SV;      // doubles per plane
  static constexpr int VBUF = 2 * PLANE;     // doubles per vector buffer (re plane, im plane)
  static constexpr size_t BLOCKS = (size_t)NSLOT * BB * 16;
  static constexpr size_t VEC = (size_t)(TW ? 3 : 2) * VBUF * 8;
  static constexpr size_t RHS = (size_t)NRHS * NC * RS * RELB;
  static constexpr size_t YRING = (size_t)RY * NCW * 32 * 16;
  static constexpr size_t BARS = 8 * (2 * NSLOT + 2);
  static constexpr size_t smem_bytes() { return BLOCKS + VEC + RHS + YRING + BARS; }
};

template <int B, int NC, bool CPLX_IN, bool TW>
__global__ void __launch_bounds__(SplitShape<B, NC, CPLX_IN, TW>::NTHR, (B == 16 && !CPLX_IN) ? 3 : 1)
    bt_sweep_split_kernel(BtSweepArgs a) {
  using Sh = SplitShape<B, NC, CPLX_IN, TW>;
  constexpr int MT = Sh::MT, KQ = Sh::KQ, NCW = Sh::NCW, NSLOT = Sh::NSLOT, NRHS = Sh::NRHS, RY = Sh::RY;
  constexpr int SV = Sh::SV, RS = Sh::RS, RELB = Sh::RELB, BB = Sh::BB, PLANE = Sh::PLANE, VBUF = Sh::VBUF;
  constexpr int NMID = TW ? 3 : 2;
  constexpr int CT = NCW * 32;
  using True = std::true_type;
  using False = std::false_type;
  const int s = blockIdx.y;
  const int half = TW ? (int)(blockIdx.x & 1) : 0;
  const int cb = (int)(TW ? blockIdx.x >> 1 : blockIdx.x);
  const int c0 = cb * NC;
  const int L = a.L, m = a.m, ldv = a.ldv;
  const int kmid = TW ? a.kmid : L - 1;
  const int H = half == 0 ? kmid : L - 1 - kmid;  // forward steps (= backward steps)
  const int nsteps = 2 * H + 1;
  const int dl = half == 0 ? 1 : -1;              // layer step of the forward half
  const int l0 = half == 0 ? 0 : L - 1;           // first forward layer
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* Blk = reinterpret_cast<double2*>(smem_raw);               // NSLOT x (B x B), swizzled rows
  double* Vs = reinterpret_cast<double*>(Blk + (size_t)NSLOT * BB);  // buffers 0, 1 [, Xb]
  double* Xb = Vs + 2 * VBUF;                                         // TW: the partner's last forward vector
  unsigned char* rhs = reinterpret_cast<unsigned char*>(Vs + (TW ? 3 : 2) * VBUF);
  double* yring = reinterpret_cast<double*>(rhs + Sh::RHS);           // [RY][2][CT]
  uint64_t* full = reinterpret_cast<uint64_t*>(yring + Sh::YRING / 8);
  uint64_t* empty = full + NSLOT;
  uint64_t* xbar = empty + NSLOT;   // TW: the partner's NCW arrivals after its Xb stores
  uint64_t* midbar = xbar + 1;      // TW && CPLX_IN: the bottom passed its middle step

  // slot s = node * chunks + chunk (chunks == 1: the node's whole chain)
  const int node = s / a.chunks;
  const size_t row0 = (size_t)(s % a.chunks) * L * B;
  const bool spike = a.chunks > 1;
  const double2* sinv = a.sinv + (size_t)s * L * BB;
  const double2* hm = a.h + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  double2* W = a.w + (size_t)node * ldv * m + row0;

  for (int i = tid; i < (int)((Sh::VEC + Sh::RHS) / 8); i += blockDim.x) Vs[i] = 0.0;  // (columns past m stay 0)
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NCW);
    }
    mbar_init(xbar, NCW);
    mbar_init(midbar, NCW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (TW) cg::this_cluster().sync();  // barriers initialised before any remote arrival

  if (warp == NCW) {  // ===================== producer warp =====================
    // One warp, kept to a few dozen instructions per step (its serial instruction latency must
    // stay well under a chain step): all pointers advance incrementally, every lane spins on the
    // slot's "empty" barrier itself (no warp sync to broadcast the wait), lane 0 issues the
    // bulk copies, and the right-hand-side tile is 16-byte cp.async pieces spread over the lanes.
    const int ncols = m - c0 < NC ? m - c0 : NC;
    constexpr int PPC = B * RELB / 16;         // 16-byte pieces per right-hand-side column
    constexpr int NP = (NC * PPC + 31) / 32;   // pieces per lane
    constexpr uint32_t BLKB = (uint32_t)(BB * 16);
    const unsigned char* rbase = CPLX_IN ? reinterpret_cast<const unsigned char*>(W)
                                         : reinterpret_cast<const unsigned char*>(a.y + row0);
    const unsigned char* rsrc[NP];  // this lane's pieces of layer l0's rows
    uint32_t rdst[NP];              // ... and their place in tile 0 (shared-memory address)
    bool rok[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int c = lane + 32 * k, col = c / PPC, pc = c % PPC;
      rok[k] = col < ncols;
      rsrc[k] = rbase + ((size_t)l0 * B + (size_t)(c0 + (rok[k] ? col : 0)) * ldv) * RELB + pc * 16;
      rdst[k] = smem_u32(rhs) + (uint32_t)(col * RS * RELB + pc * 16);
    }
    const ptrdiff_t rstep = (ptrdiff_t)dl * B * RELB;   // bytes per forward layer
    constexpr uint32_t TILEB = (uint32_t)(NC * RS * RELB);
    const uint32_t full0 = smem_u32(full), blk0 = smem_u32(Blk);
    int ps = 0, round = 0;  // ring slot to fill next, and how often the ring has wrapped
    uint32_t rt = 0;        // byte offset of the step's right-hand-side tile
    auto wait_empty = [&]() {
      if (round > 0) mbar_spin(empty + ps, (round - 1) & 1);
    };
    auto advance = [&]() {
      if (++ps == NSLOT) {
        ps = 0;
        ++round;
      }
    };
    auto copy_block = [&](const double2* src) {  // lane 0; src == nullptr: an empty slot of the step
      const uint32_t bar = full0 + 8u * ps;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(src ? BLKB : 0u) : "memory");
      if (src)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         blk0 + BLKB * ps),
                     "l"(src), "r"(BLKB), "r"(bar)
                     : "memory");
    };
    auto copy_rhs = [&](ptrdiff_t layer_off) {   // all lanes: tile rt <- the rows at rsrc + layer_off, tracked by full[ps]
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (rok[k])
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(rdst[k] + rt), "l"(rsrc[k] + layer_off));
      asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(full0 + 8u * ps) : "memory");
      __syncwarp();  // every lane's pending-count increment precedes lane 0's arrival below
      rt = rt + TILEB == NRHS * TILEB ? 0u : rt + TILEB;
    };
    // forward steps r = 0 .. H-1 on layer l = l0 + dl r: [S_l^{-1} | H], H_l = hm[l - 1] (top) or hm[l] (bottom)
    const double2* psv = sinv + (size_t)l0 * BB;
    const double2* ph = hm + ((ptrdiff_t)l0 - (half == 0 ? 1 : 0)) * BB;
    const ptrdiff_t bstep = (ptrdiff_t)dl * BB;
    ptrdiff_t roff = 0;
#pragma unroll 1
    for (int v = 0; v < H; ++v) {
      wait_empty();
      copy_rhs(roff);
      if (lane == 0) copy_block(psv);
      advance();
      wait_empty();
      if (lane == 0) copy_block(v > 0 ? ph : nullptr);
      advance();
      psv += bstep;
      ph += bstep;
      roff += rstep;
    }
    {  // middle: [T^{-1} | T^{-1} C_{k-1} | T^{-1} C_k^T] and the rows of layer kmid
      wait_empty();
      copy_rhs(((ptrdiff_t)kmid - l0) * B * RELB);
      if (lane == 0) copy_block(sinv + (size_t)kmid * BB);
      advance();
      wait_empty();
      if (lane == 0) copy_block(H > 0 ? hm + (size_t)(kmid - 1) * BB : nullptr);
      advance();
      if (TW) {
        wait_empty();
        if (lane == 0) copy_block(hm + (size_t)kmid * BB);
        advance();
      }
    }
    // backward steps rb = 0 .. H-1 on layer l = l0 + dl (H-1-rb): G = gm[l] (top) or gm[l - 1] (bottom)
    const double2* pg = gm + ((ptrdiff_t)l0 + (ptrdiff_t)dl * (H - 1) - (half == 0 ? 0 : 1)) * BB;
#pragma unroll 1
    for (int rb = 0; rb < H; ++rb) {
      wait_empty();
      if (lane == 0) copy_block(pg);
      advance();
      pg -= bstep;
    }
    return;
  }

  // ===================== compute warps =====================
  const int part = warp & 1, wt = warp >> 1;
  const double sgn = part ? 1.0 : -1.0;
  const int arow = 8 * (wt % MT) + g;
  const int aoff = t4 * B + (arow ^ (2 * t4));  // swizzle: row r of column k at r ^ 2(k & 3)
  const int bcol = 8 * (wt / MT) + g;
  const int cl0 = 8 * (wt / MT) + 2 * t4;       // this lane's output columns cl0, cl0 + 1 (row arow)
  const int vx = part * PLANE + bcol * SV + t4;        // B operand of the P chain in a vector buffer
  const int vy = (1 - part) * PLANE + bcol * SV + t4;  // ... of the Q chain
  const int vo = part * PLANE + cl0 * SV + arow;       // this lane's outputs (second column at + SV)
  const bool ok0 = c0 + cl0 < m, ok1 = c0 + cl0 + 1 < m;
  // this lane's component of W at (row arow of layer 0, column c0 + cl0); the next column at + 2 ldv
  double* const wbase = reinterpret_cast<double*>(W + arow + (size_t)(ok0 ? c0 + cl0 : 0) * ldv) + part;
  const ptrdiff_t wcol = ok1 ? 2 * (ptrdiff_t)ldv : 0;

  auto bar_step = [&]() { asm volatile("bar.sync 1, %0;\n" ::"n"(CT) : "memory"); };
  auto yslot = [&](int u) { return yring + (u & (RY - 1)) * 2 * CT + tid; };  // components at [0], [CT]
  static_assert((RY & (RY - 1)) == 0, "RY must be a power of two");
  // y_l of backward step u comes from W (cp.async, issued RY - 1 steps ahead) unless the forward
  // step that produced it is too recent (rb <= (RY - 3) / 2), in which case that step wrote the slot
  constexpr int NDIRECT = (RY - 3) / 2 + 1;  // backward steps rb = 0 .. NDIRECT - 1
  auto issue_y = [&](int u) {
    if (u >= H + 1 + NDIRECT && u < nsteps && !(a.dbg & 8)) {
      const double* gp = wbase + (ptrdiff_t)(l0 + dl * (2 * H - u)) * (2 * B);
      double* sl = yslot(u);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sl)), "l"(gp), "r"(ok0 ? 8 : 0));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sl + CT)), "l"(gp + wcol),
                   "r"(ok1 ? 8 : 0));
    }
    cp_async_commit();
  };

  // accumulators: [k-step parity] x {P, Q} x {c0, c1}
  double accP[2][2], accQ[2][2], nxtP[2][2], nxtQ[2][2];
  double2 af[KQ];   // A fragments of the dependent product of the current step
  int qs = 0, qpar = 0;  // ring slot (and its phase parity) of the next step to prepare
  int cs = 0;            // first ring slot of the current step
  int rt = 0;            // right-hand-side tile of the next step to prepare
  double* Vcur = Vs;            // buffer step v writes
  double* Vprv = Vs + VBUF;     // buffer step v - 1 wrote

  auto adv_q = [&](int n) {
    qs += n;
    if (qs >= NSLOT) {
      qs -= NSLOT;
      qpar ^= 1;
    }
  };
  auto load_af = [&](int slot) {
    const double2* Ab = Blk + (size_t)slot * BB + aoff;
#pragma unroll
    for (int q = 0; q < KQ; ++q) af[q] = Ab[4 * q * B];
  };
  auto zero_next = [&]() {
#pragma unroll
    for (int p = 0; p < 2; ++p) nxtP[p][0] = nxtP[p][1] = nxtQ[p][0] = nxtQ[p][1] = 0.0;
  };
  // next accumulators = S^{-1} Y from block `slot` and right-hand-side tile rt
  auto rhs_mma = [&](int slot) {
    if (CPLX_IN) {
      const double2* Ab = Blk + (size_t)slot * BB + aoff;
      const double* bp = reinterpret_cast<const double*>(rhs) + ((size_t)rt * NC * RS + bcol * RS + t4) * 2;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const double2 av = Ab[4 * q * B];
        dmma884(nxtP[q & 1][0], nxtP[q & 1][1], av.x, bp[8 * q + part]);
        dmma884(nxtQ[q & 1][0], nxtQ[q & 1][1], av.y, bp[8 * q + 1 - part]);
      }
    } else {
      const double* Ac = reinterpret_cast<const double*>(Blk + (size_t)slot * BB + aoff) + part;
      const double* bp = reinterpret_cast<const double*>(rhs) + (size_t)rt * NC * RS + bcol * RS + t4;
#pragma unroll
      for (int q = 0; q < KQ; ++q) dmma884(nxtP[q & 1][0], nxtP[q & 1][1], Ac[8 * q * B], bp[4 * q]);
    }
    if (++rt == NRHS) rt = 0;
  };
  // prepare a forward or middle step: blocks [S^{-1} | H] in slots qs, qs + 1 (same phase)
  const bool dbg_nowait = a.dbg & 4, dbg_noy = a.dbg & 8, dbg_noepi = a.dbg & 16;
  auto pre_fwd = [&]() {
    if (!dbg_nowait) {
    mbar_spin(full + qs, qpar);
    mbar_spin(full + qs + 1, qpar);
    }
    zero_next();
    rhs_mma(qs);
    load_af(qs + 1);
    adv_q(2);
  };
  // prepare a backward step: block G in slot qs
  auto pre_bwd = [&]() {
    if (!dbg_nowait) mbar_spin(full + qs, qpar);
    zero_next();
    load_af(qs);
    adv_q(1);
  };
  auto take_next = [&]() {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      accP[p][0] = nxtP[p][0];
      accP[p][1] = nxtP[p][1];
      accQ[p][0] = nxtQ[p][0];
      accQ[p][1] = nxtQ[p][1];
    }
  };
  // acc += M u (u: a negated running vector, two planes)
  auto vec_mma = [&](const double* Vb) {
    double bx[KQ], by[KQ];
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      bx[q] = Vb[vx + 4 * q];
      by[q] = Vb[vy + 4 * q];
    }
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      dmma884(accP[q & 1][0], accP[q & 1][1], af[q].x, bx[q]);
      dmma884(accQ[q & 1][0], accQ[q & 1][1], af[q].y, by[q]);
    }
  };
  auto fold = [&](double& r0, double& r1) {
    r0 = fma(sgn, accQ[0][0] + accQ[1][0], accP[0][0] + accP[1][0]);
    r1 = fma(sgn, accQ[0][1] + accQ[1][1], accP[0][1] + accP[1][1]);
  };
  auto release = [&](int slot, int n) {
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < n; ++i) mbar_arrive(empty + (slot + i < NSLOT ? slot + i : slot + i - NSLOT));
    }
  };
  auto swap_buffers = [&]() {
    double* t = Vcur;
    Vcur = Vprv;
    Vprv = t;
  };

  // deferred epilogue of step u (its negated x is in the buffer `Vb`, complete after the next
  // step barrier): element i = tid + k CT -> (row i % B, column i / B), coalesced column stores
  constexpr int EPT = (B * NC + CT - 1) / CT;
  const double2 coeff = a.coeff[node];
  double* const T = a.complex_mode ? nullptr : a.t + (size_t)node * ldv * m + row0;
  int eo_v[EPT];      // element offset inside a vector plane
  size_t eo_g[EPT];   // element offset in T / W without the layer term
  bool eo_ok[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int i = tid + k * CT;
    eo_v[k] = (i / B) * SV + (i % B);
    eo_ok[k] = i < B * NC && c0 + i / B < m;
    eo_g[k] = (size_t)(i % B) + (size_t)(eo_ok[k] ? c0 + i / B : 0) * ldv;
  }
  auto epi_load = [&](const double* Vb, double2 (&ex)[EPT]) {
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (eo_ok[k]) ex[k] = make_double2(Vb[eo_v[k]], Vb[PLANE + eo_v[k]]);
  };
  auto epi_store = [&](int l, const double2 (&ex)[EPT]) {
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      if (eo_ok[k]) {
        const size_t o = eo_g[k] + (size_t)l * B;
        const double2 x = make_double2(-ex[k].x, -ex[k].y);
        if (a.complex_mode) {
          W[o] = x;
        } else {
          T[o] = coeff.x * x.x - coeff.y * x.y;
          if (spike && (l == 0 || l == L - 1)) W[o] = x;  // boundary layers: x for the reduced system
        }
      }
    }
  };

  // ---------------- prologue ----------------
#pragma unroll
  for (int u = 0; u < RY - 1; ++u) issue_y(u);
  cs = qs;
  pre_fwd();
  take_next();

  // ---------------- forward steps ----------------
  // TAIL steps (the last NDIRECT, and the very last with the twisted exchange) hand y to the
  // backward half through the lane's ring slot instead of W
  auto fwd_step = [&](int v, auto tail_c) {
    constexpr bool TAIL = decltype(tail_c)::value;
    if (v > 0) {
      bar_step();
      vec_mma(Vprv);
    }
    release(cs, 2);
    issue_y(v + RY - 1);
    cs = qs;
    pre_fwd();
    double y0, y1;
    fold(y0, y1);
    take_next();
    Vcur[vo] = -y0;
    Vcur[vo + SV] = -y1;
    if (TAIL) {
      const bool last = v == H - 1;
      if (TW && last) {  // the partner's middle step needs this vector
        double* px = cg::this_cluster().map_shared_rank(Xb, half ^ 1);
        px[vo] = -y0;
        px[vo + SV] = -y1;
      }
      double* sl = yslot(2 * H - v);  // backward step H + 1 + rb, rb = H - 1 - v
      sl[0] = y0;
      sl[CT] = y1;
      if (TW && last) {
        asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(xbar, half ^ 1);
      }
    } else {
      double* wp = wbase + (ptrdiff_t)(l0 + dl * v) * (2 * B);
      if (ok0 && !dbg_noy) wp[0] = y0;
      if (ok1 && !dbg_noy) wp[wcol] = y1;
    }
    swap_buffers();
  };
  const int tail0 = H - NDIRECT > 0 ? H - NDIRECT : 0;
#pragma unroll 1
  for (int v = 0; v < tail0; ++v) fwd_step(v, False{});
#pragma unroll 1
  for (int v = tail0; v < H; ++v) fwd_step(v, True{});

  // ---------------- middle layer ----------------
  {
    const int v = H;
    if (H > 0) bar_step();
    if (TW) mbar_wait_cluster(xbar, 0);
    if (H > 0 || TW) vec_mma(TW && half == 1 ? Xb : Vprv);  // y_{k-1}
    if (TW) {
      mbar_spin(full + qs, qpar);
      load_af(qs);
      adv_q(1);
      vec_mma(half == 1 ? Vprv : Xb);                        // u_{k+1}
    }
    release(cs, NMID);
    issue_y(v + RY - 1);
    if (v + 1 < nsteps) {
      cs = qs;
      pre_bwd();
    }
    double x0, x1;
    fold(x0, x1);
    take_next();
    if (TW && CPLX_IN) {  // W row k holds the RHS both CTAs read; the top overwrites it with x_k
      if (half == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(midbar, 0);
      } else {
        mbar_wait_cluster(midbar, 0);
      }
    }
    Vcur[vo] = -x0;
    Vcur[vo + SV] = -x1;
    swap_buffers();
  }

  // ---------------- backward steps ----------------
  int le = kmid;  // layer of the step whose epilogue is pending (the middle, then the backward layers)
#pragma unroll 1
  for (int v = H + 1; v < nsteps; ++v) {
    double2 ex[EPT];
    bar_step();
    const bool ep = v > H + 1 || half == 0;
    if (ep) epi_load(Vprv, ex);
    vec_mma(Vprv);
    release(cs, 1);
    if (ep && !dbg_noepi) epi_store(le, ex);
    issue_y(v + RY - 1);
    if (v + 1 < nsteps) {
      cs = qs;
      pre_bwd();
    }
    cp_async_wait<RY - 1>();
    const double* sl = yslot(v);
    const double y0 = sl[0], y1 = sl[CT];
    double r0, r1;
    fold(r0, r1);
    take_next();
    Vcur[vo] = -(y0 + r0);
    Vcur[vo + SV] = -(y1 + r1);
    swap_buffers();
    le = l0 + dl * (2 * H - v);
  }
  cp_async_wait<0>();
  if (nsteps > 1 || half == 0) {
    double2 ex[EPT];
    bar_step();
    epi_load(Vprv, ex);
    epi_store(le, ex);
  }
}

template <int B, int NC, bool TW>
static cudaError_t launch_split(const BtSweepArgs& a0, cudaStream_t st) {
  BtSweepArgs a = a0;
  if (const char* e = getenv("FEAST_SPLIT_DBG")) a.dbg = atoi(e);
  using Sh = SplitShape<B, NC, false, TW>;
  const size_t sm = a.complex_mode ? SplitShape<B, NC, true, TW>::smem_bytes() : Sh::smem_bytes();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.m + NC - 1) / NC * (TW ? 2 : 1)), (unsigned)a.nodes);
  cfg.blockDim = dim3(Sh::NTHR);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = TW ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (a.complex_mode) {
    auto kern = bt_sweep_split_kernel<B, NC, true, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  } else {
    auto kern = bt_sweep_split_kernel<B, NC, false, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// b = 16: 8 columns per CTA on 4 compute warps + the producer warp
cudaError_t bt_sweep_split16(const BtSweepArgs& a, cudaStream_t st) {
  return a.kmid >= 0 ? launch_split<16, 8, true>(a, st) : launch_split<16, 8, false>(a, st);
}

}  // namespace feastgpu
