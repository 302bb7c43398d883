// sweep_small.cu — the block-Thomas sweep for small blocks (b = 16, 32) with a bulk-copy
// pipeline. Same recursion, twisted variant and epilogue as sweep.cu's bt_sweep_kernel:
//   forward : y_l = S_l^{-1} Y_l - H_l y_{l-1}          (the top half; the bottom half runs the
//   middle  : x_k = T^{-1} Y_k - (T^{-1}C_{k-1}) y_{k-1} [- (T^{-1}C_k^T) u_{k+1}]   same code on
//   backward: x_l = y_l - G_l x_{l+1}                    reversed layers)
//   epilogue: T = Re(c x) (real mode) or W = x (complex mode, the ShiftSystem shim)
// What changes is the data movement, which the ncu profile of the cp.async version showed
// dominating at b = 16 (DMMA 6.7% of issued instructions, the rest per-element address
// arithmetic of the producer, executed by every thread at every step):
//   * the factor blocks are stored with a row swizzle (row i of column k at i ^ 2(k & 3),
//     blocktri.cu), so each block is ONE cp.async.bulk into a conflict-free stage; one
//     producer thread issues the 1-3 copies of a step NSTAGE steps ahead, completing on the
//     stage's "full" mbarrier; compute warps release stages on "empty" mbarriers;
//   * the right-hand-side rows (Y_l forward, y_l backward) go straight to registers: each
//     lane loads the B-operand fragments it will use two steps ahead (no shared-memory slots,
//     no copies to issue); the backward's y_l fragment is exactly what this lane stored in
//     the forward, so no cross-thread ordering is involved;
//   * the running vector is double-buffered in shared memory; the compute warps synchronise
//     per step on an mbarrier (arrive after storing their rows, wait only before reading the
//     neighbour vector, so the S^{-1} Y half of a forward step runs before the wait);
//   * twisted pairs swap their last forward vectors through DSMEM and a remote mbarrier
//     arrival (no cluster-wide barrier, the producer never joins).

#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "mbarrier.cuh"

namespace cg = cooperative_groups;

namespace feastgpu {

#ifndef FEAST_SWEEP_SPIN
#define FEAST_SWEEP_SPIN 1
#endif
constexpr bool kSpin = FEAST_SWEEP_SPIN;

template <int B, int NC, int TPW, bool TW, bool CPLX_IN>
struct SmallShape {
  // pipeline depth: 3 stages. Deeper rings (5) measured no faster at b = 16 and cost the
  // occupancy the 8-column shape needs (3 CTAs per SM on config 2)
  static constexpr int NSTAGE = 3;
  // vector fragments run FD steps ahead: the backward's second step reads y written by the
  // forward step 2 + 2*1 steps earlier, so FD <= 3 (ring of FD + 1 lane-private slots)
  static constexpr int FD = NSTAGE - 1 < 3 ? NSTAGE - 1 : 3;
  static constexpr int KMAX = (TW ? 3 : 2) * B;  // stage columns (the middle step)
  static constexpr int SV = B + 4;                // running vector [col][k] stride (double2)
  static constexpr int MT = B / 8;
  static constexpr int NWARPS = MT * (NC / 8) / TPW;
  static constexpr int KQ = B / 4;
  // lane-private ring of vector fragments, NSTAGE slots: forward TPW x KQ values (8 B real,
  // 16 B complex), backward TPW x 2 complex
  static constexpr int FWDB = TPW * KQ * (CPLX_IN ? 16 : 8), BWDB = TPW * 32;
  static constexpr int SLOTB = FWDB > BWDB ? FWDB : BWDB;
  static constexpr size_t smem_bytes() {
    return sizeof(double2) * ((size_t)(TW ? 3 : 2) * NC * SV + (size_t)NSTAGE * KMAX * B) +
           (size_t)(FD + 1) * NWARPS * 32 * SLOTB + 8 * (2 * NSTAGE + 4);
  }
};

template <int B, int NC, int TPW, bool CPLX_IN, bool TW>
__global__ void __launch_bounds__((SmallShape<B, NC, TPW, TW, CPLX_IN>::NWARPS + 1) * 32)
    bt_sweep_bulk_kernel(BtSweepArgs a) {
  using Sh = SmallShape<B, NC, TPW, TW, CPLX_IN>;
  constexpr int SLOTB = Sh::SLOTB, FD = Sh::FD;
  constexpr int NSTAGE = Sh::NSTAGE, KMAX = Sh::KMAX, SV = Sh::SV, MT = Sh::MT, NWARPS = Sh::NWARPS;
  constexpr int KQ = B / 4;  // k-steps of one b x b block
  constexpr size_t BB = (size_t)B * B;
  const int s = blockIdx.y;
  const int half = TW ? (int)(blockIdx.x & 1) : 0;
  const int c0 = (int)(TW ? blockIdx.x >> 1 : blockIdx.x) * NC;
  const int L = a.L, m = a.m, ldv = a.ldv;
  const int kmid = TW ? a.kmid : L - 1;
  const int H = half == 0 ? kmid : L - 1 - kmid;  // forward steps (= backward steps)
  const int nsteps = 2 * H + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  extern __shared__ __align__(128) double2 smem[];
  double2* St = smem;                              // NSTAGE x (KMAX x B), swizzled rows
  double2* Vs0 = St + NSTAGE * KMAX * B;           // running vector, double-buffered [col][k]
  double2* Vs1 = Vs0 + NC * SV;
  double2* Xb = Vs1 + NC * SV;                     // TW: the partner's last forward vector
  char* ring = reinterpret_cast<char*>(Xb + (TW ? NC * SV : 0));  // (FD+1) x (NWARPS*32) x SLOTB
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)(FD + 1) * NWARPS * 32 * SLOTB);
  uint64_t* empty = full + NSTAGE;
  uint64_t* stepbar = empty + NSTAGE;  // NWARPS arrivals per step
  uint64_t* xbar = stepbar + 1;        // TW: the partner's NWARPS arrivals after its Xb stores
  uint64_t* midbar = xbar + 1;         // TW && CPLX_IN: the bottom passed its middle step
  // slot s = node * chunks + chunk (chunks == 1: the node's whole chain)
  const int node = s / a.chunks;
  const size_t row0 = (size_t)(s % a.chunks) * L * B;  // the chunk's first row in the node's blocks
  const bool spike = a.chunks > 1;
  const double2 coeff = a.coeff[node];
  const double2* sinv = a.sinv + (size_t)s * L * BB;
  const double2* hm = a.h + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  double2* W = a.w + (size_t)node * ldv * m + row0;
  double* T = a.complex_mode ? nullptr : a.t + (size_t)node * ldv * m + row0;
  const double* Yin = a.y ? a.y + row0 : nullptr;
  auto layer_of = [&](int r) { return half == 0 ? r : L - 1 - r; };

  for (int i = tid; i < 2 * NC * SV; i += blockDim.x) Vs0[i] = make_double2(0.0, 0.0);
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NWARPS);
    }
    mbar_init(stepbar, NWARPS);
    mbar_init(xbar, NWARPS);
    mbar_init(midbar, NWARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (TW) cg::this_cluster().sync();  // barriers initialised before any remote arrival

  if (warp == NWARPS) {  // ===================== producer =====================
    if (lane == 0) {
      for (int v = 0; v < nsteps; ++v) {
        const int st = v % NSTAGE, n = v / NSTAGE;
        if (n > 0) {
          if (kSpin) mbar_spin(empty + st, (n - 1) & 1);
          else mbar_wait(empty + st, (n - 1) & 1);
        }
        double2* dst = St + st * KMAX * B;
        const double2* src[3] = {nullptr, nullptr, nullptr};
        if (v < H) {            // forward step r = v: [S_l^{-1} | H_l]
          const int l = layer_of(v);
          src[0] = sinv + (size_t)l * BB;
          if (v > 0) src[1] = hm + (size_t)(half == 0 ? l - 1 : l) * BB;
        } else if (v == H) {    // middle: [T^{-1} | T^{-1} C_{k-1} | T^{-1} C_k^T]
          src[0] = sinv + (size_t)kmid * BB;
          if (H > 0) src[1] = hm + (size_t)(kmid - 1) * BB;
          if (TW) src[2] = hm + (size_t)kmid * BB;
        } else {                // backward: G
          const int l = layer_of(H - 1 - (v - H - 1));
          src[0] = gm + (size_t)(half == 0 ? l : l - 1) * BB;
        }
        const uint32_t nb = (src[0] != nullptr) + (src[1] != nullptr) + (src[2] != nullptr);
        mbar_expect_tx(full + st, nb * (uint32_t)(BB * 16));
#pragma unroll
        for (int i = 0; i < 3; ++i)
          if (src[i]) bulk_copy(dst + i * BB, src[i], (uint32_t)(BB * 16), full + st);
      }
    }
    return;
  }

  // ===================== compute warps =====================
  int arow[TPW], bcol[TPW], aoff[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tt = warp * TPW + j;  // TPW == MT: the warp owns whole columns (all B rows)
    arow[j] = 8 * (tt % MT) + g;
    aoff[j] = t4 * B + (arow[j] ^ (2 * t4));  // swizzle: row r of column k at r ^ 2(k & 3)
    bcol[j] = 8 * (tt / MT) + g;
  }
  // vector fragments, NSTAGE - 1 steps ahead, into this lane's slot of the ring (cp.async:
  // nothing waits until the step that reads them; each lane copies exactly what it reads)
  //   forward / middle: the RHS rows of the layer, B-fragment (k = 4q + t4, column bcol)
  //   backward        : y_l at (arow, cl0) and (arow, cl0 + 1), stored by this lane
  auto slot = [&](int v) { return ring + ((size_t)(v % (FD + 1)) * NWARPS * 32 + tid) * SLOTB; };
  auto issue_frag = [&](int v) {
    if (v < nsteps) {
      char* sl = slot(v);
      if (v <= H) {
        const int l = v < H ? layer_of(v) : kmid;
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const int gc = c0 + bcol[j];
          const bool ok = gc < m;
          const size_t base = (size_t)l * B + t4 + (size_t)(ok ? gc : 0) * ldv;
#pragma unroll
          for (int q = 0; q < KQ; ++q) {
            const uint32_t sa = smem_u32(sl + (j * KQ + q) * (CPLX_IN ? 16 : 8));
            if (CPLX_IN)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(W + base + 4 * q),
                           "r"(ok ? 16 : 0));
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(Yin + base + 4 * q),
                           "r"(ok ? 8 : 0));
          }
        }
      } else if (v > H + 1) {  // (the first backward step reads the running buffer)
        const int l = layer_of(H - 1 - (v - H - 1));
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
          const int cl = c0 + bcol[j] - g + 2 * t4;
          const size_t row = (size_t)l * B + arow[j];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = cl + e < m;
            const uint32_t sa = smem_u32(sl + (j * 2 + e) * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                         "l"(W + row + (size_t)(ok ? cl + e : 0) * ldv), "r"(ok ? 16 : 0));
          }
        }
      }
    }
    cp_async_commit();
  };
  struct FragRef {
    const char* p;
    FEAST_DEV double re(int j, int q) const { return reinterpret_cast<const double*>(p)[j * KQ + q]; }
    FEAST_DEV double2 cx(int j, int q) const { return reinterpret_cast<const double2*>(p)[j * KQ + q]; }
    FEAST_DEV double2 y(int j, int e) const { return reinterpret_cast<const double2*>(p)[j * 2 + e]; }
  };
  using Frag = FragRef;

  // accumulators: two sets by k-step parity, each split into the (a.re * b) and (a.im * b)
  // halves of the complex product, so a step's dependent DMMA chain is KQ / 2 long
  CAcc acc[TPW], acc2[TPW], accy[TPW], accy2[TPW];
  auto zero_acc = [&]() {
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      acc[j].zero();
      acc2[j].zero();
      accy[j].zero();
      accy2[j].zero();
    }
  };
  auto fold_acc = [&]() {
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      acc[j].r0 += acc2[j].r0 + (accy[j].r0 + accy2[j].r0);
      acc[j].r1 += acc2[j].r1 + (accy[j].r1 + accy2[j].r1);
      acc[j].i0 += acc2[j].i0 + (accy[j].i0 + accy2[j].i0);
      acc[j].i1 += acc2[j].i1 + (accy[j].i1 + accy2[j].i1);
    }
  };
  // (cx + cy) += a * b with the a.re and a.im products in separate accumulators
  auto cmma_split = [&](CAcc& cx, CAcc& cy, double2 av, double2 bv) {
    dmma884(cx.r0, cx.r1, av.x, bv.x);
    dmma884(cy.r0, cy.r1, -av.y, bv.y);
    dmma884(cx.i0, cx.i1, av.x, bv.y);
    dmma884(cy.i0, cy.i1, av.y, bv.x);
  };
  // acc += S x (RHS fragment): block 0 of the stage
  auto mma_rhs = [&](const double2* As, const Frag& f) {
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      CAcc* ac = (q & 1) ? acc2 : acc;
      CAcc* ay = (q & 1) ? accy2 : accy;
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const double2 av = As[4 * q * B + aoff[j]];
        if (CPLX_IN) {
          cmma_split(ac[j], ay[j], av, f.cx(j, q));
        } else {
          const double yv = f.re(j, q);
          dmma884(ac[j].r0, ac[j].r1, av.x, yv);
          dmma884(ay[j].i0, ay[j].i1, av.y, yv);
        }
      }
    }
  };
  // acc -= M x vec: block `blk` of the stage against a running vector in shared memory
  auto mma_vec = [&](const double2* As, int blk, const double2* Bv) {
    const double2* Ab = As + blk * BB;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      CAcc* ac = (q & 1) ? acc2 : acc;
      CAcc* ay = (q & 1) ? accy2 : accy;
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const double2 av = Ab[4 * q * B + aoff[j]];
        cmma_split(ac[j], ay[j], make_double2(-av.x, -av.y), Bv[bcol[j] * SV + 4 * q + t4]);
      }
    }
  };
  auto acquire = [&](int v) -> const double2* {
    if (std::is_same<decltype(a), BtSweepArgs>::value && kSpin) mbar_spin(full + v % NSTAGE, (v / NSTAGE) & 1);
    else mbar_wait(full + v % NSTAGE, (v / NSTAGE) & 1);
    return St + (v % NSTAGE) * KMAX * B;
  };
  auto release = [&](int v) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + v % NSTAGE);
  };
  // step exchange among the compute warps: a named hardware barrier (id 1; the producer never
  // joins) at the point where a warp first reads the neighbour vector, so every warp has
  // stored its rows of step v - 1 (and finished reading the buffer step v overwrites)
  auto step_arrive = [&]() {};
  auto step_wait = [&](int v) {
    if (v > 0) {
      if constexpr (TPW == MT) __syncwarp();  // the running vector's columns are this warp's own
      else asm volatile("bar.sync 1, %0;\n" ::"n"(NWARPS * 32) : "memory");
    }
  };
  auto buf = [&](int v) { return (v & 1) ? Vs1 : Vs0; };
  auto epilogue = [&](int l, int j, double2 x0, double2 x1) {
    const size_t row = (size_t)l * B + arow[j];
    const int col = c0 + bcol[j] - g + 2 * t4;
    if (a.complex_mode) {
      if (col < m) W[row + (size_t)col * ldv] = x0;
      if (col + 1 < m) W[row + (size_t)(col + 1) * ldv] = x1;
    } else {
      if (col < m) T[row + (size_t)col * ldv] = coeff.x * x0.x - coeff.y * x0.y;
      if (col + 1 < m) T[row + (size_t)(col + 1) * ldv] = coeff.x * x1.x - coeff.y * x1.y;
      if (spike && (l == 0 || l == L - 1)) {  // the chunk's boundary layers: x for the reduced system
        if (col < m) W[row + (size_t)col * ldv] = x0;
        if (col + 1 < m) W[row + (size_t)(col + 1) * ldv] = x1;
      }
    }
  };

  // one chain step v (forward v < H, middle v == H, backward v > H) on the fragments `cur`
  // loaded two steps earlier; it first issues the loads of step v + 2 into `ahead` (the
  // three fragment sets rotate by unrolling, so no register move waits on an in-flight load)
  auto step = [&](int v) {
    issue_frag(v + FD);
    cp_async_wait<FD>();  // this lane's fragments of step v have landed
    const FragRef cur{slot(v)};
    const double2* As = acquire(v);
    zero_acc();
    double2* Vout = buf(v);
    if (v < H) {  // ---------------- forward ----------------
      const int r = v, l = layer_of(r);
      mma_rhs(As, cur);
      if (r > 0) {
        step_wait(v);
        mma_vec(As, 1, buf(v - 1));
      }
      release(v);
      fold_acc();
      const bool last = r == H - 1;
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int cl0 = bcol[j] - g + 2 * t4;
        const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
        const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
        Vout[(cl0 + 0) * SV + arow[j]] = y0;
        Vout[(cl0 + 1) * SV + arow[j]] = y1;
        if (TW && last) {  // the partner's middle step needs this vector
          double2* px = cg::this_cluster().map_shared_rank(Xb, half ^ 1);
          px[(cl0 + 0) * SV + arow[j]] = y0;
          px[(cl0 + 1) * SV + arow[j]] = y1;
        }
        if (!last) {  // re-read by this lane in the backward half
          const size_t row = (size_t)l * B + arow[j];
          if (c0 + cl0 < m) W[row + (size_t)(c0 + cl0) * ldv] = y0;
          if (c0 + cl0 + 1 < m) W[row + (size_t)(c0 + cl0 + 1) * ldv] = y1;
        }
      }
      step_arrive();
      if (TW && last) {
        asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(xbar, half ^ 1);
      }
    } else if (v == H) {  // ---------------- middle layer ----------------
      mma_rhs(As, cur);
      if (H > 0) step_wait(v);
      if (TW) mbar_wait_cluster(xbar, 0);
      const double2* own = buf(v - 1);
      if (H > 0 || TW) mma_vec(As, 1, TW && half == 1 ? Xb : own);  // y_{k-1}
      if (TW) mma_vec(As, 2, half == 1 ? own : Xb);                 // u_{k+1}
      release(v);
      fold_acc();
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
        const int cl0 = bcol[j] - g + 2 * t4;
        const double2 x0 = make_double2(acc[j].r0, acc[j].i0);
        const double2 x1 = make_double2(acc[j].r1, acc[j].i1);
        Vout[(cl0 + 0) * SV + arow[j]] = x0;
        Vout[(cl0 + 1) * SV + arow[j]] = x1;
        if (half == 0) epilogue(kmid, j, x0, x1);
      }
      step_arrive();
    } else {  // ---------------- backward ----------------
      const int rb = v - H - 1, l = layer_of(H - 1 - rb);
      step_wait(v);
      mma_vec(As, 0, buf(v - 1));
      release(v);
      fold_acc();
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int cl0 = bcol[j] - g + 2 * t4;
        double2 y0, y1;
        if (rb == 0) {  // own last forward vector, same lane and element
          y0 = Vout[(cl0 + 0) * SV + arow[j]];
          y1 = Vout[(cl0 + 1) * SV + arow[j]];
        } else {
          y0 = cur.y(j, 0);
          y1 = cur.y(j, 1);
        }
        const double2 x0 = make_double2(y0.x + acc[j].r0, y0.y + acc[j].i0);
        const double2 x1 = make_double2(y1.x + acc[j].r1, y1.y + acc[j].i1);
        Vout[(cl0 + 0) * SV + arow[j]] = x0;
        Vout[(cl0 + 1) * SV + arow[j]] = x1;
        epilogue(l, j, x0, x1);
      }
      step_arrive();
    }
  };

#pragma unroll
  for (int v = 0; v < FD; ++v) issue_frag(v);
#pragma unroll 1
  for (int v = 0; v < nsteps; ++v) step(v);
  cp_async_wait<0>();
}

template <int B, int NC, int TPW, bool TW>
static cudaError_t launch_bulk(const BtSweepArgs& a, cudaStream_t st) {
  using Sh = SmallShape<B, NC, TPW, TW, false>;
  const size_t sm = a.complex_mode ? SmallShape<B, NC, TPW, TW, true>::smem_bytes() : Sh::smem_bytes();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.m + NC - 1) / NC * (TW ? 2 : 1)), (unsigned)a.nodes);
  cfg.blockDim = dim3((Sh::NWARPS + 1) * 32);
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
    auto kern = bt_sweep_bulk_kernel<B, NC, TPW, true, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  } else {
    auto kern = bt_sweep_bulk_kernel<B, NC, TPW, false, TW>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int B, int NC, int TPW>
static cudaError_t launch_bulk_any(const BtSweepArgs& a, cudaStream_t st) {
  return a.kmid >= 0 ? launch_bulk<B, NC, TPW, true>(a, st) : launch_bulk<B, NC, TPW, false>(a, st);
}

bool bt_swizzled_factors(int b) { return b == 16 || b == 32; }

// b = 16, 32 (factors in the swizzled layout, bt_swizzled_factors)
cudaError_t bt_sweep_small(const BtSweepArgs& a, cudaStream_t st) {
  switch (a.b) {
    case 16:  // sweep_pipe.cu: 8 columns per CTA, software-pipelined steps, lean producer warp
      return bt_sweep_pipe16(a, st);
    case 32:  // (complex right-hand sides: narrower column blocks keep the ring within 227 KB)
      return a.complex_mode ? launch_bulk_any<32, 8, 1>(a, st) : launch_bulk_any<32, 16, 1>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
