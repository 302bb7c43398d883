// sweep_pipe.cu — the block-Thomas sweep for b = 16 (config 2's storage): software-pipelined
// chain steps, one warp per 8-row tile.
//
// Same recursion, twisted variant, SPIKE chunk slots and epilogue as sweep_small.cu:
//   forward : y_l = S_l^{-1} Y_l - H_l y_{l-1}
//   middle  : x_k = T^{-1} Y_k - (T^{-1}C_{k-1}) y_{k-1} [- (T^{-1}C_k^T) u_{k+1}]
//   backward: x_l = y_l - G_l x_{l+1}
//   epilogue: T = Re(c x) (real mode) or W = x (complex mode)
//
// What the ncu captures of the earlier b = 16 kernels showed (profiles/r02_cfg2_full.ncu-rep,
// profiles/r02_sweep_split_v3.ncu-rep) and what this kernel does about it:
//   * the single producer thread was the pacemaker: ~150 dependent instructions per step of
//     address arithmetic kept it from running ahead of the chain. Here every pointer and ring
//     position advances incrementally, all lanes spin on the slot's "empty" barrier themselves,
//     lane 0 issues the block copies and the right-hand-side tile is 16-byte cp.async pieces
//     spread over the lanes (tracked by the same mbarrier);
//   * shared-memory bandwidth is as scarce as the FP64 pipe (an m8n8k4 DMMA needs a 256-byte A
//     and a 256-byte B fragment): each warp computes a full complex 8 x 8 tile, so one 16-byte
//     A load and one 16-byte B load feed four DMMAs (2 wavefronts per DMMA; splitting the real
//     and imaginary parts over two warps, tried first, needs 4 and ran into the shared pipe);
//   * the step is software-pipelined: everything of step v + 1 that does not depend on the
//     running vector (waiting for its factor blocks, the S^{-1} Y product, loading the A
//     fragments of the dependent product) is issued behind step v's dependent DMMAs, before
//     step v's result is folded and stored, so only  barrier -> vector loads -> 16 DMMAs ->
//     fold -> store  remains on the chain. The running vector is kept NEGATED (u = -y), so the
//     chain accumulates acc += M u with the A fragments as loaded, and the only sign is at the
//     fold: re = P - Q (P = a.re u.re, Q = a.im u.im), im = P' + Q';
//   * factor blocks travel in a ring of single-block slots (a forward step takes two, a
//     backward step one); the backward's y_l comes back through a lane-private cp.async ring
//     RY - 1 steps ahead (each lane re-reads exactly what it stored; the last forward steps hand
//     their y over in shared memory);
//   * shared-memory layouts are conflict-free for both the C-fragment stores and the
//     B-fragment loads (rows XOR-swizzled by the column).

#include <cooperative_groups.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "mbarrier.cuh"

namespace cg = cooperative_groups;

namespace feastgpu {

template <int B, int NC, bool CPLX_IN, bool TW>
struct PipeShape {
  static constexpr int MT = B / 8, NT = NC / 8, KQ = B / 4;
  // row tiles per compute warp: all of them for b = 16 (one warp owns a column tile's whole chain:
  // no block barrier per step, each B fragment feeds both row tiles)
  static constexpr int TPW = 1;
  static constexpr int NCW = MT * NT / TPW;  // compute warps
  // warps of a CTA take consecutive hardware warp slots and slot % 4 picks the SM sub-partition:
  // pad the CTA to 3 warps (compute, producer, idle) so the compute warps of the 3 CTAs of an SM
  // land on different sub-partitions (slots 0, 3, 6)
  static constexpr int NIDLE = NCW == 1 ? 1 : 0;
  static constexpr int NTHR = (NCW + 1 + NIDLE) * 32;
  static constexpr int NSLOT = 10;           // factor-block ring (even: a forward step takes 2)
  static constexpr int NRHS = NSLOT / 2;     // right-hand-side tiles, one per forward step in flight
  static constexpr int RY = 8;               // lane-private y ring (backward), RY - 1 steps ahead
  static constexpr int SV = B + 4;           // running vector [col][k] stride (double2)
  static constexpr int RS = B + 4;           // right-hand-side tile [col][k] stride (elements)
  static constexpr int RELB = CPLX_IN ? 16 : 8;
  static constexpr int BB = B * B;
  static constexpr int VBUF = NC * SV;       // double2 per vector buffer
  static constexpr size_t BLOCKS = (size_t)NSLOT * BB * 16;
  static constexpr size_t VEC = (size_t)(TW ? 3 : 2) * VBUF * 16;
  static constexpr size_t RHS = (size_t)NRHS * NC * RS * RELB;
  static constexpr size_t YRING = (size_t)RY * 2 * TPW * NCW * 32 * 16;
  static constexpr size_t BARS = 8 * (2 * NSLOT + 2);
  static constexpr size_t smem_bytes() { return BLOCKS + VEC + RHS + YRING + BARS; }
};

template <int B, int NC, bool CPLX_IN, bool TW>
__global__ void __launch_bounds__(PipeShape<B, NC, CPLX_IN, TW>::NTHR, (B == 16 && !CPLX_IN) ? 3 : 1)
    bt_sweep_pipe_kernel(BtSweepArgs a) {
  using Sh = PipeShape<B, NC, CPLX_IN, TW>;
  constexpr int MT = Sh::MT, KQ = Sh::KQ, NCW = Sh::NCW, TPW = Sh::TPW, NSLOT = Sh::NSLOT, NRHS = Sh::NRHS, RY = Sh::RY;
  constexpr int SV = Sh::SV, RS = Sh::RS, RELB = Sh::RELB, BB = Sh::BB, VBUF = Sh::VBUF;
  constexpr int NMID = TW ? 3 : 2;
  constexpr int CT = NCW * 32;
  using True = std::true_type;
  using False = std::false_type;
  const int s = blockIdx.y;
  const int half = TW ? (int)(blockIdx.x & 1) : 0;
  const int c0 = (int)(TW ? blockIdx.x >> 1 : blockIdx.x) * NC;
  const int L = a.L, m = a.m, ldv = a.ldv;
  const int kmid = TW ? a.kmid : L - 1;
  const int H = half == 0 ? kmid : L - 1 - kmid;  // forward steps (= backward steps)
  const int nsteps = 2 * H + 1;
  const int dl = half == 0 ? 1 : -1;              // layer step of the forward half
  const int l0 = half == 0 ? 0 : L - 1;           // first forward layer
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* Blk = reinterpret_cast<double2*>(smem_raw);   // NSLOT x (B x B), swizzled rows
  double2* Vs = Blk + (size_t)NSLOT * BB;                // buffers 0, 1 [, Xb]: element (c, r) at c SV + (r ^ (c & 6))
  double2* Xb = Vs + 2 * VBUF;                           // TW: the partner's last forward vector
  unsigned char* rhs = reinterpret_cast<unsigned char*>(Vs + (TW ? 3 : 2) * VBUF);
  double2* yring = reinterpret_cast<double2*>(rhs + Sh::RHS);  // [RY][2][CT]
  uint64_t* full = reinterpret_cast<uint64_t*>(yring + Sh::YRING / 16);
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

  {  // zero the vectors and the right-hand-side tiles (columns past m stay 0)
    double* z = reinterpret_cast<double*>(Vs);
    for (int i = tid; i < (int)((Sh::VEC + Sh::RHS) / 8); i += blockDim.x) z[i] = 0.0;
  }
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

  if (warp > NCW) return;  // idle padding warps
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
  // warp wt owns row tiles wt % (MT / TPW) * TPW + j (j < TPW) of column tile wt / (MT / TPW)
  constexpr int WPC = MT / TPW;  // warps per column tile
  const int wt = warp;
  const int ntile = wt / WPC;
  int arow[TPW], aoff[TPW], vo[TPW];
  const int bcol = 8 * ntile + g;
  const int cl0 = 8 * ntile + 2 * t4;           // this lane's output columns cl0, cl0 + 1
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    arow[j] = 8 * ((wt % WPC) * TPW + j) + g;
    aoff[j] = t4 * B + (arow[j] ^ (2 * t4));    // factor blocks: row r of column k at r ^ 2(k & 3)
    vo[j] = cl0 * SV + (arow[j] ^ (cl0 & 6));   // this lane's outputs (second column at + SV)
  }
  // B fragment of k-step q: vector element (c = bcol, r = 4q + t4) at c SV + (r ^ (c & 6))
  //   = bcol SV + (t4 ^ (bcol & 2)) + 4 (q ^ sw), sw = (bcol >> 2) & 1
  const int sw4 = 4 * ((bcol >> 2) & 1);
  const int vb_e = bcol * SV + (t4 ^ (bcol & 2)) + sw4;  // even q: + 4q
  const int vb_o = bcol * SV + (t4 ^ (bcol & 2)) - sw4;  // odd q : + 4q
  const uint32_t ok0 = c0 + cl0 < m, ok1 = c0 + cl0 + 1 < m;
  // W and T at (row g of layer 0, column c0 + cl0); row tile j at + 8 j, the next column at + wcol
  double2* const wbase = W + arow[0] + (size_t)(ok0 ? c0 + cl0 : 0) * ldv;
  const ptrdiff_t wcol = ok1 ? (ptrdiff_t)ldv : 0;
  const double2 coeff = a.coeff[node];
  double* const tbase =
      CPLX_IN ? nullptr : a.t + (size_t)node * ldv * m + row0 + arow[0] + (size_t)(ok0 ? c0 + cl0 : 0) * ldv;
  const ptrdiff_t lstep = (ptrdiff_t)dl * B;  // elements per forward layer step

  auto bar_step = [&]() {
    if (NCW == 1) __syncwarp();
    else asm volatile("bar.sync 1, %0;\n" ::"n"(CT) : "memory");
  };
  // lane-private y ring: element (step u, row tile j, column e) at ((u % RY) (2 TPW) + 2 j + e) CT + tid
  auto yslot = [&](int u) { return yring + (u & (RY - 1)) * 2 * TPW * CT + tid; };
  static_assert((RY & (RY - 1)) == 0, "RY must be a power of two");
  // y_l of backward step u comes from W (cp.async, issued RY - 1 steps ahead) unless the forward
  // step that produced it is too recent (rb <= (RY - 3) / 2), in which case that step wrote the slot
  constexpr int NDIRECT = (RY - 3) / 2 + 1;  // backward steps rb = 0 .. NDIRECT - 1
  // the cp.async source of backward step u: layer l0 + dl (2H - u); it moves by -lstep per step
  const double2* yp = wbase + (ptrdiff_t)(l0 + dl * (2 * H - (RY - 1))) * B;  // for u = RY - 1 (first in-loop issue)
  auto issue_y = [&](int u) {  // called with u = v + RY - 1 for v = 0, 1, ... (yp follows)
    if (u >= H + 1 + NDIRECT && u < nsteps) {
      double2* sl = yslot(u);
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sl + (2 * j) * CT)),
                     "l"(yp + 8 * j), "r"(ok0 ? 16 : 0));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sl + (2 * j + 1) * CT)),
                     "l"(yp + 8 * j + wcol), "r"(ok1 ? 16 : 0));
      }
    }
    cp_async_commit();
    yp -= lstep;
  };

  // accumulators [k-step parity][output column]: re = Pr - Qr, im = Pi + Qi with
  //   Pr += a.re u.re, Qr += a.im u.im, Pi += a.re u.im, Qi += a.im u.re
  struct Acc {
    double pr[2][2], qr[2][2], pi[2][2], qi[2][2];
    FEAST_DEV void zero() {
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int e = 0; e < 2; ++e) pr[p][e] = qr[p][e] = pi[p][e] = qi[p][e] = 0.0;
    }
  };
  Acc acc[TPW], nxt[TPW];
  double2 af[TPW][KQ];   // A fragments of the dependent product of the current step
  int qs = 0, qpar = 0;  // ring slot (and its phase parity) of the next step to prepare
  int cs = 0;            // first ring slot of the current step
  int rt = 0;            // right-hand-side tile of the next step to prepare
  double2* Vcur = Vs;          // buffer step v writes
  double2* Vprv = Vs + VBUF;   // buffer step v - 1 wrote

  auto adv_q = [&](int n) {
    qs += n;
    if (qs >= NSLOT) {
      qs -= NSLOT;
      qpar ^= 1;
    }
  };
  // the phase check of a "full" barrier costs ~90 clocks even when the phase is complete, so it is
  // issued ahead of the dependent DMMAs (test) and only consumed behind them (wait)
  auto test = [&](int slot) -> uint32_t {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(full + slot)), "r"((uint32_t)qpar)
        : "memory");
    return ok;
  };
  auto wait = [&](int slot, uint32_t ok) {
    if (!ok) mbar_spin(full + slot, qpar);
  };
  auto load_af = [&](int slot) {
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const double2* Ab = Blk + (size_t)slot * BB + aoff[j];
#pragma unroll
      for (int q = 0; q < KQ; ++q) af[j][q] = Ab[4 * q * B];
    }
  };
  // next accumulators = S^{-1} Y from block `slot` and right-hand-side tile rt
  auto rhs_mma = [&](int slot) {
#pragma unroll
    for (int j = 0; j < TPW; ++j) nxt[j].zero();
    if (CPLX_IN) {
      const double2* bp = reinterpret_cast<const double2*>(rhs) + (size_t)rt * NC * RS + bcol * RS + t4;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const double2 bv = bp[4 * q];
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const double2 av = Blk[(size_t)slot * BB + aoff[j] + 4 * q * B];
          dmma884(nxt[j].pr[q & 1][0], nxt[j].pr[q & 1][1], av.x, bv.x);
          dmma884(nxt[j].qr[q & 1][0], nxt[j].qr[q & 1][1], av.y, bv.y);
          dmma884(nxt[j].pi[q & 1][0], nxt[j].pi[q & 1][1], av.x, bv.y);
          dmma884(nxt[j].qi[q & 1][0], nxt[j].qi[q & 1][1], av.y, bv.x);
        }
      }
    } else {
      const double* bp = reinterpret_cast<const double*>(rhs) + (size_t)rt * NC * RS + bcol * RS + t4;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const double yv = bp[4 * q];
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const double2 av = Blk[(size_t)slot * BB + aoff[j] + 4 * q * B];
          dmma884(nxt[j].pr[q & 1][0], nxt[j].pr[q & 1][1], av.x, yv);
          dmma884(nxt[j].qi[q & 1][0], nxt[j].qi[q & 1][1], av.y, yv);
        }
      }
    }
    if (++rt == NRHS) rt = 0;
  };
  // acc += M u (u: a negated running vector)
  auto load_b = [&](const double2* Vb, double2 (&bv)[KQ]) {
#pragma unroll
    for (int q = 0; q < KQ; ++q) bv[q] = Vb[((q & 1) ? vb_o : vb_e) + 4 * q];
  };
  auto vec_mma = [&](const double2 (&bv)[KQ]) {
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        dmma884(acc[j].pr[q & 1][0], acc[j].pr[q & 1][1], af[j][q].x, bv[q].x);
        dmma884(acc[j].qr[q & 1][0], acc[j].qr[q & 1][1], af[j][q].y, bv[q].y);
        dmma884(acc[j].pi[q & 1][0], acc[j].pi[q & 1][1], af[j][q].x, bv[q].y);
        dmma884(acc[j].qi[q & 1][0], acc[j].qi[q & 1][1], af[j][q].y, bv[q].x);
      }
    }
  };
  // the NEGATED result: -re = Q - P, -im = -(P' + Q')
  auto fold_neg = [&](const Acc& c, double2& n0, double2& n1) {
    n0.x = (c.qr[0][0] + c.qr[1][0]) - (c.pr[0][0] + c.pr[1][0]);
    n0.y = -(c.pi[0][0] + c.pi[1][0]) - (c.qi[0][0] + c.qi[1][0]);
    n1.x = (c.qr[0][1] + c.qr[1][1]) - (c.pr[0][1] + c.pr[1][1]);
    n1.y = -(c.pi[0][1] + c.pi[1][1]) - (c.qi[0][1] + c.qi[1][1]);
  };
  auto release = [&](int slot, int n) {
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < n; ++i) mbar_arrive(empty + (slot + i < NSLOT ? slot + i : slot + i - NSLOT));
    }
  };
  auto swap_buffers = [&]() {
    double2* t = Vcur;
    Vcur = Vprv;
    Vprv = t;
  };
  // predicated stores (no divergent branch around a two-instruction body)
  auto st_c = [&](double2* p, double2 v, uint32_t ok) {
    asm volatile("{\n.reg .pred P1;\nsetp.ne.u32 P1, %3, 0;\n@P1 st.global.v2.f64 [%0], {%1, %2};\n}\n" ::"l"(p),
                 "d"(v.x), "d"(v.y), "r"(ok)
                 : "memory");
  };
  auto st_r = [&](double* p, double v, uint32_t ok) {
    asm volatile("{\n.reg .pred P1;\nsetp.ne.u32 P1, %2, 0;\n@P1 st.global.f64 [%0], %1;\n}\n" ::"l"(p), "d"(v),
                 "r"(ok)
                 : "memory");
  };
  // epilogue of row tile j from the negated x; wp / tp: this lane's W / T element of the layer (row tile 0)
  auto epilogue = [&](double2* wp, double* tp, int j, bool boundary, double2 n0, double2 n1) {
    if (CPLX_IN) {
      st_c(wp + 8 * j, make_double2(-n0.x, -n0.y), ok0);
      st_c(wp + 8 * j + wcol, make_double2(-n1.x, -n1.y), ok1);
    } else {
      st_r(tp + 8 * j, coeff.y * n0.y - coeff.x * n0.x, ok0);
      st_r(tp + 8 * j + wcol, coeff.y * n1.y - coeff.x * n1.x, ok1);
      if (boundary) {  // SPIKE: the chunk's boundary layers keep x for the reduced system
        st_c(wp + 8 * j, make_double2(-n0.x, -n0.y), ok0);
        st_c(wp + 8 * j + wcol, make_double2(-n1.x, -n1.y), ok1);
      }
    }
  };

  // ---------------- prologue ----------------
#pragma unroll
  for (int u = 0; u < RY - 1; ++u) cp_async_commit();  // (no backward step is that early: empty groups)
  cs = qs;
  mbar_spin(full + qs, qpar);
  mbar_spin(full + qs + 1, qpar);
  rhs_mma(qs);
  load_af(qs + 1);
  adv_q(2);
#pragma unroll
  for (int j = 0; j < TPW; ++j) acc[j] = nxt[j];

  // ---------------- forward steps ----------------
  // TAIL steps (the last NDIRECT, and the very last with the twisted exchange) hand y to the
  // backward half through the lane's ring slot instead of W
  double2* wp = wbase + (ptrdiff_t)l0 * B;  // this lane's W element of the forward layer
  auto fwd_step = [&](int v, auto tail_c) {
    constexpr bool TAIL = decltype(tail_c)::value;
    uint32_t t0, t1;
    if (v > 0) {
      double2 bv[KQ];
      bar_step();
      load_b(Vprv, bv);
      t0 = test(qs);
      t1 = test(qs + 1);
      vec_mma(bv);
    } else {
      t0 = test(qs);
      t1 = test(qs + 1);
    }
    release(cs, 2);
    issue_y(v + RY - 1);
    cs = qs;
    wait(qs, t0);
    wait(qs + 1, t1);
    rhs_mma(qs);          // step v + 1 (forward or middle): S^{-1} Y into nxt
    load_af(qs + 1);
    adv_q(2);
    const bool last = v == H - 1;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      double2 n0, n1;
      fold_neg(acc[j], n0, n1);
      acc[j] = nxt[j];
      Vcur[vo[j]] = n0;
      Vcur[vo[j] + SV] = n1;
      const double2 y0 = make_double2(-n0.x, -n0.y), y1 = make_double2(-n1.x, -n1.y);
      if (TAIL) {
        if (TW && last) {  // the partner's middle step needs this vector
          double2* px = cg::this_cluster().map_shared_rank(Xb, half ^ 1);
          px[vo[j]] = n0;
          px[vo[j] + SV] = n1;
        }
        double2* sl = yslot(2 * H - v);  // backward step H + 1 + rb, rb = H - 1 - v
        sl[(2 * j) * CT] = y0;
        sl[(2 * j + 1) * CT] = y1;
      } else {
        st_c(wp + 8 * j, y0, ok0);
        st_c(wp + 8 * j + wcol, y1, ok1);
      }
    }
    if (TAIL && TW && last) {
      asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(xbar, half ^ 1);
    }
    wp += lstep;
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
    double2 bv[KQ];
    if (H > 0) bar_step();
    if (TW) mbar_wait_cluster(xbar, 0);
    if (H > 0 || TW) {
      load_b(TW && half == 1 ? Xb : Vprv, bv);  // y_{k-1}
      vec_mma(bv);
    }
    if (TW) {
      mbar_spin(full + qs, qpar);
      load_af(qs);
      adv_q(1);
      load_b(half == 1 ? Vprv : Xb, bv);         // u_{k+1}
      vec_mma(bv);
    }
    release(cs, NMID);
    issue_y(v + RY - 1);
    if (v + 1 < nsteps) {
      cs = qs;
      mbar_spin(full + qs, qpar);
      load_af(qs);
      adv_q(1);
    }
    if (TW && CPLX_IN) {  // W row k holds the RHS both CTAs read; the top overwrites it with x_k
      if (half == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(midbar, 0);
      } else {
        mbar_wait_cluster(midbar, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      double2 n0, n1;
      fold_neg(acc[j], n0, n1);
      Vcur[vo[j]] = n0;
      Vcur[vo[j] + SV] = n1;
      if (half == 0)
        epilogue(wbase + (ptrdiff_t)kmid * B, CPLX_IN ? nullptr : tbase + (ptrdiff_t)kmid * B, j,
                 spike && (kmid == 0 || kmid == L - 1), n0, n1);
    }
    swap_buffers();
  }

  // ---------------- backward steps ----------------
  // (a chunk's boundary layers 0 and L - 1 are the last backward steps of the two halves)
  double2* ewp = wbase + (ptrdiff_t)(l0 + dl * (H - 1)) * B;
  double* etp = CPLX_IN ? nullptr : tbase + (ptrdiff_t)(l0 + dl * (H - 1)) * B;
#pragma unroll 1
  for (int v = H + 1; v < nsteps; ++v) {
    double2 bv[KQ];
    bar_step();
    load_b(Vprv, bv);
    const bool more = v + 1 < nsteps;
    const uint32_t t0 = more ? test(qs) : 1u;
#pragma unroll
    for (int j = 0; j < TPW; ++j) acc[j].zero();
    vec_mma(bv);
    release(cs, 1);
    issue_y(v + RY - 1);
    if (more) {
      cs = qs;
      wait(qs, t0);
      load_af(qs);
      adv_q(1);
    }
    cp_async_wait<RY - 1>();
    const double2* sl = yslot(v);
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const double2 y0 = sl[(2 * j) * CT], y1 = sl[(2 * j + 1) * CT];
      double2 n0, n1;
      fold_neg(acc[j], n0, n1);
      n0.x -= y0.x;   // -(y + r)
      n0.y -= y0.y;
      n1.x -= y1.x;
      n1.y -= y1.y;
      Vcur[vo[j]] = n0;
      Vcur[vo[j] + SV] = n1;
      epilogue(ewp, etp, j, spike && !more, n0, n1);
    }
    ewp -= lstep;
    if (!CPLX_IN) etp -= lstep;
    swap_buffers();
  }
  cp_async_wait<0>();
}

template <int B, int NC, bool TW>
static cudaError_t launch_pipe(const BtSweepArgs& a, cudaStream_t st) {
  using Sh = PipeShape<B, NC, false, TW>;
  const size_t sm = a.complex_mode ? PipeShape<B, NC, true, TW>::smem_bytes() : Sh::smem_bytes();
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
    auto kern = bt_sweep_pipe_kernel<B, NC, true, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  } else {
    auto kern = bt_sweep_pipe_kernel<B, NC, false, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// b = 16: 8 columns per CTA, one compute warp + the producer warp
cudaError_t bt_sweep_pipe16(const BtSweepArgs& a, cudaStream_t st) {
  return a.kmid >= 0 ? launch_pipe<16, 8, true>(a, st) : launch_pipe<16, 8, false>(a, st);
}

}  // namespace feastgpu
