// tsg_tc05.cu -- the light-row SEaC numeric pass on the 5th-generation tensor
// cores (tcgen05.mma, accumulators in TMEM): the experiment of VERDICT r01
// item 4 / north_star "(3) ... tcgen05 batched over many tile pairs where
// that measures faster", measured against panel_numeric_kernel (mma.sync).
//
// Same contract as panel_numeric_kernel (tsg_panel.cu) on light rows, TENSOR
// mode, device output: per CSR row the realised entries appended in column
// order at row_stage[row], realised counts in rowcnt, counted_elements
// (structural nonzeros), filtered pairs / segments / raw pairs in stats.
// Restates per panel of 8 tile rows (M = 128):
//   enumerate_pairs / filter_zero_products   pipeline.cpp:37-70
//   counting_pass                             kernels.cpp:79-103
//   multiply_pass / finalize_segment          kernels.cpp:105-203
//
// A persistent CTA (one per SM: it owns all 512 TMEM columns) takes panels
// of 8 tile rows.  The panel's inner tile columns K (union of its A tiles)
// and output tile columns J (union of the B tile rows k in K) are sorted in
// shared memory; J is cut into windows of 16.  Per window, for every k with
// B tiles (k, J) in the window (a work item):
//   producers (warps 0-3)  densify A_k = the 8 A tiles (I, k) stacked (128 x
//                          16, zero rows where A(I, k) is absent) and the
//                          window's B tiles (k, J) into a shared-memory ring
//                          stage, in the K-major no-swizzle canonical layout,
//                          values and 0/1 indicators;
//   MMA issuer (warp 4)    per B tile two tcgen05.mma M128 N16 K16, f16 in,
//                          f32 accumulate in TMEM: values into columns
//                          16 s and indicators into 256 + 16 s (s = the J's
//                          slot in the window); tcgen05.commit frees the stage;
//   epilogue (warps 5-8)   one thread per panel row (= TMEM lane): tcgen05.ld
//                          of its 16 slots, structural = indicator != 0,
//                          realised = value != 0 appended to the row's staging.
#include <cstdint>

#include "tsg_kernels.cuh"
#include "tsg_mma.cuh"

namespace tsg {

namespace {

constexpr int kTcThreads = 288;     // 4 producer warps, 1 MMA warp, 4 epilogue warps
constexpr int kTcStages = 4;        // ring stages (one work item each; stage = producer warp)
constexpr int kTcMaxK = 256;        // 8 tile rows x <= 32 A tiles
constexpr int kTcMaxJ = 2048;       // gathered B tiles of the panel (else: fall back)
constexpr int kTcMaxItems = 256;
constexpr uint32_t kABytes = 128 * 16 * 2;   // A_k block (values), K-major canonical
constexpr uint32_t kBBytes = 16 * 16 * 2;    // one B tile (values)
constexpr uint32_t kStageBytes = 2 * kABytes + 16 * 2 * kBBytes;  // A val + ind, 16 B tiles val + ind

struct TcSmem {
  alignas(1024) uint8_t ring[kTcStages][kStageBytes];
  uint32_t kcol[kTcMaxK];          // the panel's inner tile columns (sorted)
  uint32_t ktile[kTcMaxK][8];      // A tile index of (tile row r, k), or kNoTile
  uint16_t kocc[kTcMaxK][8];       // its column occupancy (0 when absent)
  uint32_t gather[kTcMaxJ];        // sort buffer (k or J keys)
  uint32_t jcol[kTcMaxJ];          // the panel's output tile columns (sorted, unique)
  uint32_t bstart[kTcMaxK];        // per k: first B tile of the current window
  uint32_t bfirst[kTcMaxK];        // per k: its first B tile and its offset in bcolk
  uint32_t koff[kTcMaxK + 1];
  uint32_t bcolk[kTcMaxJ];         // per k (at koff), the tile columns of B row k
  uint32_t item_k[kTcMaxItems];    // window work items: index into kcol
  uint32_t item_b0[kTcMaxItems + 1];
  uint32_t bt_idx[kTcMaxItems * 16];
  uint8_t bt_slot[kTcMaxItems * 16];
  uint64_t full[kTcStages], empty[kTcStages], tfull, tempty;
  uint32_t wsum[8];
  uint32_t tmem_base;
  uint32_t nk, nj, nitems, panel, flag;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// K-major, no-swizzle canonical layout: core matrices of 8 rows x 16 bytes,
// row groups SBO = 128 B apart, the two 8-element K halves LBO apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3fffu);
  d |= uint64_t((lbo >> 4) & 0x3fffu) << 16;
  d |= uint64_t((128u >> 4) & 0x3fffu) << 32;  // SBO
  d |= uint64_t(1) << 46;                       // version (sm_100)
  return d;                                     // base offset 0, layout SWIZZLE_NONE
}
// kind::f16, D f32, A/B f16 K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, bool acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(uint32_t(acc)));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte offset of (row m, inner k) in a K-major canonical block with `rows` rows
__device__ __forceinline__ uint32_t kmaj(uint32_t m, uint32_t k, uint32_t rows) {
  return (k >> 3) * (rows * 16u) + (m >> 3) * 128u + (m & 7u) * 16u + (k & 7u) * 2u;
}

// Bitonic sort of n keys (power of two, <= kTcMaxJ) in shared memory by the
// first `nthreads` threads; padding keys are 0xffffffff.
__device__ void bitonic(uint32_t* a, uint32_t n, int tid, int nthreads, int named_bar) {
  for (uint32_t size = 2; size <= n; size <<= 1)
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < n / 2; i += nthreads) {
        const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint32_t x = a[lo], y = a[hi];
        if ((x > y) == up) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      asm volatile("bar.sync %0, %1;" ::"r"(named_bar), "r"(nthreads));
    }
}

// Exclusive scan of one u32 per thread over the first 256 threads (named
// barrier 1); returns the exclusive prefix, total in `tot`.
__device__ __forceinline__ uint32_t scan256(uint32_t x, uint32_t* wsum, int tid, uint32_t& tot) {
  const int lane = tid & 31, w = tid >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  asm volatile("bar.sync 1, 256;" ::: "memory");
  uint32_t pre = 0;
  tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t v = wsum[i];
    if (i < w) pre += v;
    tot += v;
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  return pre + inc - x;
}

}  // namespace

__global__ void __launch_bounds__(kTcThreads, 1) tc05_panel_kernel(
    TileMat A, TileMat B, int64_t rows, const uint32_t* __restrict__ row_stage, uint64_t stage_cap,
    uint2* __restrict__ stage, int64_t* __restrict__ rowcnt, unsigned long long* __restrict__ counted,
    const unsigned long long* __restrict__ need, unsigned long long* __restrict__ stats,
    const unsigned* __restrict__ gate, unsigned* __restrict__ work, unsigned* __restrict__ fallback) {
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (*need > stage_cap || (*need >> 32)) return;  // arena too small: the host reruns the pass
  if (gate && ((gate[0] & (kErrInvariant | kErrRowPtr)) || gate[1] > 32u)) return;
  const uint32_t npanels = (A.tile_rows + 7) / 8;
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&sm.full[s], 32);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tfull, 1);
    mbar_init(&sm.tempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {  // the MMA warp owns the TMEM allocation (all 512 columns)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // pipeline phases (per role, carried across windows and panels)
  uint32_t item_base = 0, win_it = 0;  // running item count (ring stage = count % 4), windows
  // epilogue state: this thread's panel row
  unsigned long long n_struct = 0, n_filt = 0, n_seg = 0, n_raw = 0;
  for (;;) {
    if (tid == 0) sm.panel = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t P = sm.panel;
    if (P >= npanels) break;
    const uint32_t I0 = P * 8;
    // ---- panel setup (first 256 threads): K = union of the panel's A tile
    // columns with, per (k, tile row r), the A tile; J = union of the B tile
    // rows k in K (sorted, unique)
    if (tid < 256) {
      const uint32_t r = uint32_t(tid) >> 5, I = I0 + r;
      uint32_t key = 0xffffffffu;
      if (I < A.tile_rows) {
        const uint32_t a0 = A.trp[I], na = A.trp[I + 1] - a0;
        uint32_t raw = 0;
        if (uint32_t(lane) < na) {
          const uint32_t k = __ldg(&A.tco[a0 + lane].x);
          key = (k << 8) | (r << 5) | uint32_t(lane);
          raw = __ldg(B.trp + k + 1) - __ldg(B.trp + k);
        }
        n_raw += raw;
      }
      sm.gather[tid] = key;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      bitonic(sm.gather, 256, tid, 256, 1);
      // unique k: heads of runs of equal k
      const uint32_t key2 = sm.gather[tid];
      const uint32_t k = key2 >> 8;
      const bool valid = key2 != 0xffffffffu;
      const bool head = valid && (tid == 0 || (sm.gather[tid - 1] >> 8) != k);
      uint32_t nk;
      const uint32_t pos = scan256(head ? 1u : 0u, sm.wsum, tid, nk);
      if (head) {
        sm.kcol[pos] = k;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          sm.ktile[pos][q] = kNoTile;
          sm.kocc[pos][q] = 0;
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid == 0) sm.nk = nk;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // A tile of (k, r): the key's run index = number of heads at or before it - 1
      {
        uint32_t dummy;
        const uint32_t incl = scan256(head ? 1u : 0u, sm.wsum, tid, dummy) + (head ? 1u : 0u);
        if (valid) {
          const uint32_t at = A.trp[I0 + ((key2 >> 5) & 7u)] + (key2 & 31u);
          sm.ktile[incl - 1][(key2 >> 5) & 7u] = at;
          sm.kocc[incl - 1][(key2 >> 5) & 7u] = uint16_t(__ldg(&A.tco[at].y) & 0xffffu);
        }
      }
      // J gather: thread i < nk writes B row kcol[i]'s tile columns
      asm volatile("bar.sync 1, 256;" ::: "memory");
      uint32_t b0 = 0, len = 0;
      if (uint32_t(tid) < nk) {
        const uint32_t kk = sm.kcol[tid];
        b0 = __ldg(B.trp + kk);
        len = __ldg(B.trp + kk + 1) - b0;
        sm.bstart[tid] = 0;
        sm.bfirst[tid] = b0;
      }
      uint32_t tot;
      const uint32_t off = scan256(len, sm.wsum, tid, tot);
      if (uint32_t(tid) < nk) sm.koff[tid] = off;
      if (tid == 0) sm.koff[nk] = tot;
      if (tot > uint32_t(kTcMaxJ)) {
        if (tid == 0) sm.flag = 1u;
      } else {
        if (tid == 0) sm.flag = 0u;
        for (uint32_t q = 0; q < len; ++q) {
          const uint32_t J = __ldg(&B.tco[b0 + q].x);
          sm.gather[off + q] = J;
          sm.bcolk[off + q] = J;
        }
        uint32_t n2 = 32;
        while (n2 < tot) n2 <<= 1;
        for (uint32_t i = tot + tid; i < n2; i += 256) sm.gather[i] = 0xffffffffu;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        bitonic(sm.gather, n2, tid, 256, 1);
        // unique J
        uint32_t nj = 0, run = 0;
        for (uint32_t base = 0; base < tot; base += 256) {
          const uint32_t i = base + tid;
          const bool h = i < tot && (i == 0 || sm.gather[i] != sm.gather[i - 1]);
          uint32_t t2;
          const uint32_t p2 = scan256(h ? 1u : 0u, sm.wsum, tid, t2);
          if (h) sm.jcol[run + p2] = sm.gather[i];
          run += t2;
        }
        nj = run;
        if (tid == 0) sm.nj = nj;
      }
    }
    __syncthreads();
    if (sm.flag) {  // too many B tiles for one panel: the host falls back to the mma.sync pass
      if (tid == 0) atomicOr(fallback, 1u);
      break;
    }
    const uint32_t nk = sm.nk;
    const uint32_t nj = sm.nj;
    uint32_t ep_cur = 0;  // epilogue: this thread's row's entries so far
    // ---- windows of 16 output tile columns
    for (uint32_t w0 = 0; w0 < nj; w0 += 16) {
      const uint32_t wn = min(16u, nj - w0);
      const uint32_t jlast = sm.jcol[w0 + wn - 1];
      if (tid < 256) {  // work items: per k (thread), its B tiles with J in the window
        uint32_t cnt = 0, b = 0, bend = 0;  // b: position within B row k (bcolk at koff)
        if (uint32_t(tid) < nk) {
          b = sm.bstart[tid];
          bend = sm.koff[tid + 1] - sm.koff[tid];
          const uint32_t* bc = sm.bcolk + sm.koff[tid];
          while (b + cnt < bend && bc[b + cnt] <= jlast) ++cnt;
        }
        uint32_t ni, nb;
        const uint32_t ip = scan256(cnt ? 1u : 0u, sm.wsum, tid, ni);
        const uint32_t bp = scan256(cnt, sm.wsum, tid, nb);
        if (cnt) {
          sm.item_k[ip] = uint32_t(tid);
          sm.item_b0[ip] = bp;
          uint32_t s2 = 0;
          for (uint32_t q = 0; q < cnt; ++q) {
            const uint32_t bt_i = sm.bfirst[tid] + b + q;
            const uint2 bt = __ldg(B.tco + bt_i);
            while (sm.jcol[w0 + s2] < bt.x) ++s2;
            sm.bt_idx[bp + q] = bt_i;
            sm.bt_slot[bp + q] = uint8_t(s2);
#pragma unroll
            for (int r = 0; r < 8; ++r)  // filtered pairs: A column occupancy & B row occupancy
              n_filt += (uint32_t(sm.kocc[tid][r]) & (bt.y >> 16)) != 0u;
          }
          sm.bstart[tid] = b + cnt;
        }
        if (tid == 0) {
          sm.item_b0[ni] = nb;
          sm.nitems = ni;
        }
      }
      __syncthreads();
      const uint32_t ni = sm.nitems;
      if (warp < 4) {
        // ---- producers: warp w densifies the items g = w (mod 4) of the running
        // item count into ring stage w (four items in flight): the item's A_k
        // block (8 tile rows, lane-dense A chunks -> K-major rows 16 r + row)
        // and its B tiles (B-role chunks hold B^T in A order, registers
        // {reg0, reg2, reg1, reg3})
        for (uint32_t it = 0; it < ni; ++it) {
          const uint32_t gi = item_base + it;
          if ((gi & 3u) != uint32_t(warp)) continue;
          const uint32_t s = gi & 3u, ph = (gi >> 2) & 1u;
          mbar_wait(&sm.empty[s], ph ^ 1u);
          uint8_t* st = sm.ring[s];
          const uint32_t ki = sm.item_k[it];
          const int g = lane >> 2, t = lane & 3;
          const unsigned lt = lanemask_lt(), bit = 1u << lane;
          uint2 am[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const uint32_t at = sm.ktile[ki][r];
            am[r] = at != kNoTile ? __ldg(A.meta[kRoleA] + at) : make_uint2(0, 0);
          }
          uint4 ach[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) ach[r] = load_chunk(A.chunk[kRoleA], am[r].x, am[r].y, lt, bit);
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const uint32_t regs[4] = {ach[r].x, ach[r].y, ach[r].z, ach[r].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {  // reg i: row g + 8(i&1), cols 2t + 8(i>>1) .. +1
              const uint32_t off = kmaj(uint32_t(16 * r + g + 8 * (i & 1)), uint32_t(2 * t + 8 * (i >> 1)), 128);
              *reinterpret_cast<uint32_t*>(st + off) = regs[i];
              *reinterpret_cast<uint32_t*>(st + kABytes + off) = nz_h2(regs[i]);
            }
          }
          const uint32_t b0 = sm.item_b0[it], b1 = sm.item_b0[it + 1];
          for (uint32_t q0 = b0; q0 < b1; q0 += 4) {
            uint2 bm[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              bm[u] = q0 + u < b1 ? __ldg(B.meta[kRoleB] + sm.bt_idx[q0 + u]) : make_uint2(0, 0);
            uint4 bch[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) bch[u] = load_chunk(B.chunk[kRoleB], bm[u].x, bm[u].y, lt, bit);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (q0 + u >= b1) break;
              const uint32_t regs[4] = {bch[u].x, bch[u].z, bch[u].y, bch[u].w};  // back to A order of B^T
              uint8_t* bv = st + 2 * kABytes + (q0 + u - b0) * 2 * kBBytes;
#pragma unroll
              for (int i = 0; i < 4; ++i) {  // B^T row n = g + 8(i&1), inner k = 2t + 8(i>>1)
                const uint32_t off = kmaj(uint32_t(g + 8 * (i & 1)), uint32_t(2 * t + 8 * (i >> 1)), 16);
                *reinterpret_cast<uint32_t*>(bv + off) = regs[i];
                *reinterpret_cast<uint32_t*>(bv + kBBytes + off) = nz_h2(regs[i]);
              }
            }
          }
          fence_proxy_async();
          mbar_arrive(&sm.full[s]);
        }
      } else if (warp == 4) {
        // ---- MMA issuer: D[slot] += A_k . B(k, J); the first MMA of a slot overwrites
        if (lane == 0) {
          mbar_wait(&sm.tempty, (win_it & 1u) ^ 1u);  // the epilogue drained the previous window
          tc_fence_after();
          uint32_t touched = 0;
          for (uint32_t it = 0; it < ni; ++it) {
            const uint32_t gi = item_base + it;
            const uint32_t s = gi & 3u, ph = (gi >> 2) & 1u;
            mbar_wait(&sm.full[s], ph);
            tc_fence_after();
            const uint32_t base = smem_u32(sm.ring[s]);
            const uint64_t a_val = smem_desc(base, 128u * 16u), a_ind = smem_desc(base + kABytes, 128u * 16u);
            const uint32_t b0 = sm.item_b0[it], b1 = sm.item_b0[it + 1];
            for (uint32_t q = b0; q < b1; ++q) {
              const uint32_t slot = sm.bt_slot[q];
              const uint32_t bb = base + 2 * kABytes + (q - b0) * 2 * kBBytes;
              const bool acc = (touched >> slot) & 1u;
              mma_f16(tmem + 16 * slot, a_val, smem_desc(bb, 16u * 16u), acc);
              mma_f16(tmem + 256 + 16 * slot, a_ind, smem_desc(bb + kBBytes, 16u * 16u), acc);
              touched |= 1u << slot;
            }
            mma_commit(&sm.empty[s]);  // the stage is free once these MMAs have read it
          }
          mma_commit(&sm.tfull);  // the window's accumulators are complete
        }
        __syncwarp();
      } else {
        // ---- epilogue: thread = panel row = TMEM lane 32 (warp % 4) + lane
        const uint32_t q4 = uint32_t(warp & 3);
        const uint32_t prow = 32 * q4 + uint32_t(lane);  // row within the panel
        const int64_t row = int64_t(I0) * 16 + prow;
        mbar_wait(&sm.tfull, win_it & 1u);
        tc_fence_after();
        uint32_t cur = ep_cur;
        const uint32_t sbase = row < rows ? __ldg(row_stage + row) : 0u;
        for (uint32_t s = 0; s < wn; ++s) {
          uint32_t v[16], ind[16];
          const uint32_t ta = tmem + ((32u * q4) << 16) + 16u * s;
          tmem_ld16(ta, v);
          tmem_ld16(ta + 256, ind);
          tmem_ld_wait();
          const uint32_t J = sm.jcol[w0 + s];
          uint32_t nst = 0;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            nst += __uint_as_float(ind[c]) != 0.0f;
            const float x = __uint_as_float(v[c]);
            if (row < rows && x != 0.0f) stage[sbase + cur++] = make_uint2(__float_as_uint(x), J * 16u + uint32_t(c));
          }
          if (row >= rows) nst = 0;
          n_struct += nst;
          // output tile (I, J) of this row's tile row exists iff any of its 16 rows is structural
          const unsigned bal = __ballot_sync(kFull, nst != 0u);
          if (lane == 0) n_seg += ((bal & 0xffffu) != 0u) + ((bal >> 16) != 0u);
        }
        ep_cur = cur;
        tc_fence_before();
        mbar_arrive(&sm.tempty);
      }
      ++win_it;
      item_base += ni;
      __syncthreads();  // the window's lists are rewritten next
    }
    if (warp >= 5) {  // realised entries of this thread's row
      const int64_t row = int64_t(I0) * 16 + 32 * (warp & 3) + lane;
      if (row < rows) rowcnt[row] = int64_t(ep_cur);
    }
    __syncthreads();
  }
  // statistics
  n_struct = __reduce_add_sync(kFull, uint32_t(n_struct));
  if (lane == 0 && n_struct) atomicAdd(counted, n_struct);
  if (stats && (n_filt | n_seg | n_raw)) {
    atomicAdd(stats, n_filt);
    atomicAdd(stats + 1, n_seg);
    atomicAdd(stats + 2, n_raw);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

size_t tc05_smem_bytes() { return sizeof(TcSmem) + 1024; }

cudaError_t launch_tc05_panel(const TileMat& A, const TileMat& B, int64_t rows, const uint32_t* row_stage,
                              uint64_t stage_cap, uint2* stage, int64_t* rowcnt, unsigned long long* counted,
                              const unsigned long long* need, unsigned long long* stats, const unsigned* gate,
                              unsigned* work, unsigned* fallback, int device, cudaStream_t st) {
  static int sms[16] = {0};
  const int d = device & 15;
  const size_t smem = tc05_smem_bytes();
  if (!sms[d]) {
    cudaError_t e = cudaFuncSetAttribute(tc05_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, device);
  }
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const uint32_t npanels = (A.tile_rows + 7) / 8;
  const unsigned grid = std::min<unsigned>(unsigned(sms[d]), std::max<uint32_t>(npanels, 1u));
  tc05_panel_kernel<<<grid, kTcThreads, smem, st>>>(A, B, rows, row_stage, stage_cap, stage, rowcnt, counted, need,
                                                    stats, gate, work, fallback);
  return cudaGetLastError();
}

}  // namespace tsg
