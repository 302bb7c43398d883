// sweep_tma.cu — the block-Thomas sweep for large blocks (b >= 128) with a warp-specialised
// bulk-copy pipeline. Same recursion and epilogue as sweep.cu (forward y_l = S_l^{-1} Y_l -
// H_l y_{l-1}, backward x_l = y_l - G_l x_{l+1}, T_e = Re(c_e x)); what changes is the
// producer:
//   * the factors are stored in row panels (kernels.h: bt_panel_rows), so one chunk of the
//     CTA's RB rows is ONE contiguous slab; one producer thread issues a single cp.async.bulk
//     per chunk (plus one per right-hand-side column at a step's first chunk) completing on
//     an mbarrier with a transaction byte count (SASS: UBLKCP), NSTAGE chunks ahead; the
//     panel rows are XOR-swizzled so the compute warps' 16-byte shared loads stay
//     conflict-free without padding;
//   * the compute warps wait on the stage's "full" mbarrier and release it on its "empty"
//     mbarrier — no block-wide barrier per chunk, no address arithmetic in compute warps;
//   * the right-hand-side rows of each step (Y_l forward, this CTA's rows of y_l backward)
//     ride the same pipeline into a ring of vector slots;
//   * rows are split over a thread-block cluster of P CTAs as in sweep.cu (DSMEM exchange of
//     each step's result), but the per-step exchange is an mbarrier with remote arrivals that
//     a warp waits on only when it next needs the running vector (forward: at the first H_l
//     chunk, so the S_l^{-1} Y_l half covers the exchange latency).

#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "mbarrier.cuh"

namespace cg = cooperative_groups;

namespace feastgpu {

template <int B, int P>
struct TmaShape {
  static constexpr int RB = B / P;
  static constexpr int KC = (B * RB * 16 <= 32 * 1024) ? B : (32 * 1024) / (RB * 16);  // columns per chunk
  static constexpr int NCHF = 2 * B / KC, NCHB = B / KC;
  static constexpr int SA = RB;      // stage column stride (double2); panel rows are swizzled
  static constexpr int SV = B + 4;   // running vector [col][k] stride (double2)
  static constexpr int SY = B + 4;   // real vector slot stride (double)
};

template <int B, int P, int NC, int TPW, int NSTAGE>
__global__ void __launch_bounds__(((B / P / 8) * (NC / 8) / TPW + 1) * 32)
    bt_sweep_tma_kernel(BtSweepArgs a) {
  using Sh = TmaShape<B, P>;
  constexpr int RB = Sh::RB, KC = Sh::KC, NCHF = Sh::NCHF, NCHB = Sh::NCHB;
  constexpr int SA = Sh::SA, SV = Sh::SV, SY = Sh::SY;
  constexpr bool VDB = B * NC <= 2048;  // double-buffered running vector
  constexpr int VSN = 2;                // vector slots (>= 8 chunks per step: the producer is < 1 step ahead)
  constexpr int SLOT = NC * SY;         // doubles per slot (real Y_l, or this CTA's rows of y_l as double2)
  constexpr int MT = RB / 8;
  constexpr int NWARPS = MT * (NC / 8) / TPW;
  constexpr bool SPLIT = TPW <= 2;
  constexpr size_t BB = (size_t)B * B;
  static_assert(NCHB >= NSTAGE, "vector slot ring assumes the producer runs < 1 step ahead");
  const int s = blockIdx.y;
  const int prank = P > 1 ? (int)(blockIdx.x % P) : 0;
  const int c0 = (blockIdx.x / P) * NC;
  const int row0 = prank * RB;
  const int L = a.L, m = a.m, ldv = a.ldv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  extern __shared__ __align__(128) double2 smem[];
  double2* Vs0 = smem;
  double2* Vs1 = VDB ? Vs0 + NC * SV : Vs0;
  double* Vslot = reinterpret_cast<double*>(Vs1 + NC * SV);  // VSN x SLOT doubles
  double2* St = reinterpret_cast<double2*>(Vslot + VSN * SLOT);
  uint64_t* full = reinterpret_cast<uint64_t*>(St + NSTAGE * KC * SA);
  uint64_t* empty = full + NSTAGE;
  uint64_t* stepbar = empty + NSTAGE;  // per-step exchange barrier: P x NWARPS arrivals
  const double2 coeff = a.coeff[s];
  const double2* sinv = a.sinv + (size_t)s * L * BB;
  const double2* hm = a.h + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  const double2* gm = a.g + (size_t)s * (L > 1 ? L - 1 : 0) * BB;
  double2* W = a.w + (size_t)s * ldv * m;
  const bool cplx_out = a.complex_mode == 2;
  double* T = cplx_out ? nullptr : a.t + (size_t)s * ldv * m;
  const int total = L * NCHF + (L - 1) * NCHB;

  for (int i = tid; i < (VDB ? 2 : 1) * NC * SV; i += blockDim.x) Vs0[i] = make_double2(0.0, 0.0);
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NWARPS);
    }
    mbar_init(stepbar, P * NWARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (P > 1) cg::this_cluster().sync();

  if (warp == NWARPS) {  // ===================== producer =====================
    if (lane == 0) {
      for (int q = 0; q < total; ++q) {
        const int st = q % NSTAGE, n = q / NSTAGE;
        if (n > 0) mbar_wait(empty + st, (n - 1) & 1);
        double2* dst = St + st * KC * SA;
        const bool fwd = q < L * NCHF;
        int l, j;
        if (fwd) {
          l = q / NCHF;
          j = q - l * NCHF;
        } else {
          const int q2 = q - L * NCHF;
          l = L - 2 - q2 / NCHB;
          j = q2 - (q2 / NCHB) * NCHB;
        }
        // bytes of this chunk (expect before issuing)
        uint32_t bytes = 0;
        int ncols = KC;
        if (fwd && l == 0 && j * KC >= B) ncols = 0;  // H_0 = 0: nothing to load
        bytes += (uint32_t)ncols * RB * 16;
        int nvec = 0;
        if (j == 0) {
          for (int col = 0; col < NC; ++col) nvec += (c0 + col < m);
          bytes += (uint32_t)nvec * (fwd ? B * 8 : RB * 16);
        }
        mbar_expect_tx(full + st, bytes);
        if (ncols) {  // one contiguous KC x RB slab of this CTA's row panel
          const int kg = j * KC;
          const size_t pan = (size_t)prank * B * RB;
          const double2* src;
          if (fwd) src = kg < B ? sinv + (size_t)l * BB + pan + (size_t)kg * RB
                                : hm + (size_t)(l - 1) * BB + pan + (size_t)(kg - B) * RB;
          else src = gm + (size_t)l * BB + pan + (size_t)kg * RB;
          bulk_copy(dst, src, KC * RB * 16, full + st);
        }
        if (j == 0) {
          const int vseq = fwd ? l : L + (L - 2 - l);
          double* vd = Vslot + (vseq % VSN) * SLOT;
          // backward: y_l was stored to W by the compute warps (generic proxy) before they
          // released an earlier stage — order it before the bulk (async proxy) read
          if (!fwd) asm volatile("fence.proxy.async.global;\n" ::: "memory");
          for (int col = 0; col < NC; ++col) {
            const int gc = c0 + col;
            if (gc >= m) continue;
            if (fwd) bulk_copy(vd + col * SY, a.y + (size_t)l * B + (size_t)gc * ldv, B * 8, full + st);
            else bulk_copy(reinterpret_cast<double2*>(vd) + col * (SY / 2), W + (size_t)l * B + row0 + (size_t)gc * ldv,
                           RB * 16, full + st);
          }
        }
      }
    }
    __syncwarp();
    if (P > 1) cluster_sync_unaligned();  // matches the compute warps' final barrier
    return;
  }

  // ===================== compute warps =====================
  int qc = 0;
  auto acquire = [&]() -> const double2* {
    mbar_wait(full + qc % NSTAGE, (qc / NSTAGE) & 1);
    return St + (qc % NSTAGE) * KC * SA;
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + qc % NSTAGE);
    ++qc;
  };
  // exchange barrier among the compute warps of the whole cluster (the producer never joins),
  // split in two: after its DSMEM stores a warp fences and arrives on every CTA's step
  // mbarrier; it waits on its own CTA's only when it next reads the running vector — the
  // forward step's S_l^{-1} Y_l half needs no y_{l-1}, so the exchange hides behind it
  uint32_t step_phase = 0;
  bool pending = false;
  auto step_arrive = [&]() {
    asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
    __syncwarp();
    if (lane < P) mbar_arrive_cluster(stepbar, lane);
    pending = true;
  };
  auto step_wait = [&]() {
    if (pending) {
      mbar_wait_cluster(stepbar, step_phase & 1);
      ++step_phase;
      pending = false;
    }
  };

  CAcc acc[TPW], acc2[SPLIT ? TPW : 1];
  int arow[TPW], grow[TPW], bcol[TPW], aoff[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tt = warp + NWARPS * j;
    arow[j] = 8 * (tt % MT) + g;
    aoff[j] = t4 * SA + (arow[j] ^ (2 * t4));  // panel swizzle: row r of column k at r ^ 2(k&3)
    grow[j] = row0 + arow[j];
    bcol[j] = 8 * (tt / MT) + g;
  }
  auto put = [&](double2* Vout, int idx, double2 val) {
    if (P == 1) {
      Vout[idx] = val;
    } else {
      cg::cluster_group cl = cg::this_cluster();
#pragma unroll
      for (int q = 0; q < P; ++q) cl.map_shared_rank(Vout, q)[idx] = val;
    }
  };
  auto zero_acc = [&]() {
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      acc[j].zero();
      if (SPLIT) acc2[j].zero();
    }
  };
  auto fold_acc = [&]() {
    if (SPLIT) {
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        acc[j].r0 += acc2[j].r0; acc[j].r1 += acc2[j].r1;
        acc[j].i0 += acc2[j].i0; acc[j].i1 += acc2[j].i1;
      }
    }
  };

  // ---------------- forward sweep ----------------
  for (int l = 0; l < L; ++l) {
    const double2* Bv = (l & 1) ? Vs0 : Vs1;  // y_{l-1}
    double2* Vout = (l & 1) ? Vs1 : Vs0;
    const double* Ys = Vslot + (l % VSN) * SLOT;
    zero_acc();
#pragma unroll 1
    for (int c = 0; c < NCHF; ++c) {
      if (c * KC == B) step_wait();  // first H_l chunk: y_{l-1} from the whole cluster
      const double2* As = acquire();
      if (!(l == 0 && c * KC >= B)) {
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
          const int kg = c * KC + kk;  // warp-uniform
          CAcc* ac = (SPLIT && ((kk >> 2) & 1)) ? acc2 : acc;
          if (kg < B) {
#pragma unroll
            for (int j = 0; j < TPW; ++j) {
              const double2 av = As[kk * SA + aoff[j]];
              const double yv = Ys[bcol[j] * SY + kg + t4];
              dmma884(ac[j].r0, ac[j].r1, av.x, yv);
              dmma884(ac[j].i0, ac[j].i1, av.y, yv);
            }
          } else {
#pragma unroll
            for (int j = 0; j < TPW; ++j) {
              const double2 av = As[kk * SA + aoff[j]];
              cmma(ac[j], make_double2(-av.x, -av.y), Bv[bcol[j] * SV + kg - B + t4]);
            }
          }
        }
      }
      release();
    }
    fold_acc();
    if (!VDB) {  // single running buffer: everyone is done with y_{l-1}
      step_arrive();
      step_wait();
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      const double2 y0 = make_double2(acc[j].r0, acc[j].i0);
      const double2 y1 = make_double2(acc[j].r1, acc[j].i1);
      put(Vout, (cl0 + 0) * SV + grow[j], y0);
      put(Vout, (cl0 + 1) * SV + grow[j], y1);
      if (l + 1 < L) {
        const size_t row = (size_t)l * B + grow[j];
        if (c0 + cl0 < m) W[row + (size_t)(c0 + cl0) * ldv] = y0;
        if (c0 + cl0 + 1 < m) W[row + (size_t)(c0 + cl0 + 1) * ldv] = y1;
      }
    }
    step_arrive();
  }

  // ---------------- backward sweep ----------------
  auto epilogue = [&](int l, int j, double2 x0, double2 x1) {
    const size_t row = (size_t)l * B + grow[j];
    const int col = c0 + bcol[j] - g + 2 * t4;
    if (cplx_out) {  // x itself (its y_l rows were fetched into the slot before this step)
      if (col < m) W[row + (size_t)col * ldv] = x0;
      if (col + 1 < m) W[row + (size_t)(col + 1) * ldv] = x1;
      return;
    }
    if (col < m) T[row + (size_t)col * ldv] = coeff.x * x0.x - coeff.y * x0.y;
    if (col + 1 < m) T[row + (size_t)(col + 1) * ldv] = coeff.x * x1.x - coeff.y * x1.y;
  };
#pragma unroll
  for (int j = 0; j < TPW; ++j)
    epilogue(L - 1, j, make_double2(acc[j].r0, acc[j].i0), make_double2(acc[j].r1, acc[j].i1));

  for (int l = L - 2; l >= 0; --l) {
    const double2* Bv = (l & 1) ? Vs0 : Vs1;  // x_{l+1}
    double2* Vout = (l & 1) ? Vs1 : Vs0;
    // this CTA's rows of y_l: from the slot, except y_{L-2} (finished one step ago; its slot
    // copy may predate it) which still sits in the buffer this step writes x_{L-2} into
    const double2* Yc = reinterpret_cast<const double2*>(Vslot + ((L + (L - 2 - l)) % VSN) * SLOT);
    zero_acc();
    step_wait();  // x_{l+1} from the whole cluster
#pragma unroll 1
    for (int c = 0; c < NCHB; ++c) {
      const double2* As = acquire();
#pragma unroll
      for (int kk = 0; kk < KC; kk += 4) {
        const int kg = c * KC + kk;
        CAcc* ac = (SPLIT && ((kk >> 2) & 1)) ? acc2 : acc;
#pragma unroll
        for (int j = 0; j < TPW; ++j) cmma(ac[j], As[kk * SA + aoff[j]], Bv[bcol[j] * SV + kg + t4]);
      }
      release();
    }
    fold_acc();
    if (!VDB) {
      step_arrive();
      step_wait();
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int cl0 = bcol[j] - g + 2 * t4;
      double2 y0, y1;
      if (l == L - 2 && VDB) {
        y0 = Vout[(cl0 + 0) * SV + grow[j]];
        y1 = Vout[(cl0 + 1) * SV + grow[j]];
      } else if (l == L - 2) {  // single buffer: y_{L-2} from global (this lane wrote it)
        const size_t row = (size_t)l * B + grow[j];
        y0 = c0 + cl0 < m ? W[row + (size_t)(c0 + cl0) * ldv] : make_double2(0.0, 0.0);
        y1 = c0 + cl0 + 1 < m ? W[row + (size_t)(c0 + cl0 + 1) * ldv] : make_double2(0.0, 0.0);
      } else {
        y0 = Yc[(cl0 + 0) * (SY / 2) + arow[j]];
        y1 = Yc[(cl0 + 1) * (SY / 2) + arow[j]];
      }
      const double2 x0 = make_double2(y0.x - acc[j].r0, y0.y - acc[j].i0);
      const double2 x1 = make_double2(y1.x - acc[j].r1, y1.y - acc[j].i1);
      put(Vout, (cl0 + 0) * SV + grow[j], x0);
      put(Vout, (cl0 + 1) * SV + grow[j], x1);
      epilogue(l, j, x0, x1);
    }
    step_arrive();
  }
  if (P > 1) cluster_sync_unaligned();  // no CTA leaves while its peers may still address it
}

template <int B, int P, int NC, int TPW, int NSTAGE>
static cudaError_t launch_tma(const BtSweepArgs& a, cudaStream_t st) {
  using Sh = TmaShape<B, P>;
  constexpr int NWARPS = (B / P / 8) * (NC / 8) / TPW;
  constexpr bool VDB = B * NC <= 2048;
  const size_t sm = sizeof(double2) * (size_t)(VDB ? 2 : 1) * NC * Sh::SV + sizeof(double) * 2 * NC * Sh::SY +
                    sizeof(double2) * (size_t)NSTAGE * Sh::KC * Sh::SA + 16 * NSTAGE + 8;
  auto kern = bt_sweep_tma_kernel<B, P, NC, TPW, NSTAGE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.m + NC - 1) / NC * P), (unsigned)a.nodes);
  cfg.blockDim = dim3((NWARPS + 1) * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// launch shapes: b -> (cluster size P, panel rows RB = b / P)
int bt_panel_rows(int b) {
  switch (b) {
    case 128: return 64;
    case 256: return 128;
    case 512: return 128;
  }
  return 0;
}

// sweeps over panel-layout factors (b in {128, 256, 512}); real right-hand sides, output T
// (mode 0) or x (mode 2)
cudaError_t bt_sweep_tma(const BtSweepArgs& a, cudaStream_t st) {
  if (a.complex_mode == 1 || a.ldv % 2) return cudaErrorInvalidValue;
  switch (a.b) {
    case 128: return launch_tma<128, 2, 8, 1, 3>(a, st);
    // clusters of 2: every SM can host one (clusters of 4 leave 16 of 148 idle, GPC
    // granularity — tools/microbench/cluster_occ.cu), measured 8% faster on config 3
    case 256: return launch_tma<256, 2, 8, 2, 3>(a, st);
    case 512: return launch_tma<512, 4, 8, 2, 2>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace feastgpu
