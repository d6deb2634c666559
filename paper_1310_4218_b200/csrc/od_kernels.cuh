// sm_100a kernels of the column-update path.
//
//  jacobi_step   3D 7-point Jacobi ("laminar diffusion") over all
//                fields of all resident chunks in one launch (chunk-index
//                table), k-marching with a cp.async plane ring.  HBM-bound.
//  physics_step  the Fig. 4 column recurrence, one thread
//                per column, trip count floor(nz*C)-1 from the (shifted) load
//                multiplier field.  FP64-pipe-bound.
//  pack_faces    boundary strips of chunks that border another rank into a
//                contiguous per-peer send buffer (Fig. 2 "compute boundaries").
//  init_chunk    seeded initial state, keyed by global coordinates.
//
// All arithmetic on field values uses explicit IEEE round-to-nearest
// intrinsics so the results are bitwise equal to oracle/field_oracle.c.
#pragma once

#include <cstdint>
#include <type_traits>

namespace odb {

// Jacobi weights: u' = W1*((xm+xp)+(ym+yp)+(zm+zp)) + W0*u, W0 + 6*W1 = 1.
constexpr double kW0 = 0.25;
constexpr double kW1 = 0.125;
// physics map: y <- R*(y - y^2) + (b+1)/512 ; R = 4 - 1/64
constexpr double kR = 3.984375;
constexpr double kEps = 0.001953125;  // 2^-9

enum Face : int32_t { kLeft = 0, kRight = 1, kTop = 2, kBottom = 3 };

struct FaceDev {
  const double* p;     // element (f=0, k=0, e=0) of the strip
  int64_t fs, ks, es;  // strides (elements) for field, level, position along the face
  const double* lo;    // the allocation the strip lies in: [lo, hi) (checked builds)
  const double* hi;
  // TMA source of a top/bottom face row (full tiles): a chunk row map (tkind 0,
  // coordinates (x, trow, plane)) or a received strip's map (tkind 1, (x, plane))
  const void* tm;
  int32_t trow, tkind;
};

struct ChunkDev {
  const double* in;  // U^t, [F][nz][h][pitch]
  double* out;       // U^{t+1}
  double* a;         // physics state A, [nz][h][pitch]
  int64_t fstride;   // nz * kstride
  int64_t kstride;   // h * pitch
  int32_t w, h, pitch, x0, y0, vp;
  int32_t rmask;  // P2P halos: bit d set when face d is a strip received from a peer GPU
  int32_t pad1;
  FaceDev face[4];
  // TMA tensor maps of U^t for full tiles (null: the chunk has no full tile or
  // TMA staging is off): box tw x th x 1 (main) and tw x 1 x 1 (row)
  const void* tm_main;
  const void* tm_row;
};

struct TileDev {
  int32_t slot, tx0, ty0;
  int32_t pad;     // fused tiles: bit 0 = reads a remote strip, bits 1.. = canonical id
  int32_t tw, th;  // fused tiles: width 8/16/32/64 and height 256 / tw (4 row warps)
  int32_t lg, pad2;  // log2(tw / 2)
};
__device__ __forceinline__ int share_tag(const TileDev& t) {
  return (t.slot << 20) | (t.ty0 << 8) | (t.tx0 >> 5);
}

struct PackJob {
  int32_t slot, side, len, lenp;  // side: which edge of the source chunk; lenp: row stride
  int64_t dst;                   // element offset into the send buffer
  int32_t peer;                  // destination rank
  int32_t rflag;                 // index of the face's flag in the peer's flag array
  int64_t rdst;                  // element offset in the peer's receive buffer half
};

__device__ __forceinline__ uint64_t dmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double unit_hash(uint64_t seed, uint64_t idx) {
  return double(dmix64(seed ^ dmix64(idx)) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Checked build (libod_b200_checked.so, -DOD_CHECKED; compute-sanitizer is not
// available on the GPU pool): every walker's first and last global address is
// checked against its allocation, every shared-memory ring offset against the
// plane, and random sleeps are injected at the cross-CTA synchronisation
// points (tile step stamps, pack counters, halo flags) and inside the ring
// hand-off, so ordering bugs that a lucky schedule hides surface as wrong
// fields in the bitwise stress tests (tests/test_gpu_stress.py).
#ifdef OD_CHECKED
#define OD_CHECK(cond, what)                                                              \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("od checked: %s failed (block %d, thread %d,%d)\n", what, int(blockIdx.x),   \
             int(threadIdx.x), int(threadIdx.y));                                         \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
__device__ __forceinline__ uint64_t dmix64(uint64_t x);
__device__ __forceinline__ void od_jitter(unsigned salt) {
  const uint64_t h = dmix64(globaltimer_ns() ^ (uint64_t(blockIdx.x) << 32) ^
                            (uint64_t(threadIdx.y * 32 + threadIdx.x) << 20) ^ salt);
  if ((h & 7) == 0) __nanosleep(unsigned(h >> 40) & 8191);
}
#else
#define OD_CHECK(cond, what) \
  do {                       \
  } while (0)
__device__ __forceinline__ void od_jitter(unsigned) {}
#endif
__device__ __forceinline__ bool od_in(const double* p, const double* lo, const double* hi) {
  return p >= lo && p < hi;
}

// Per-SM processor-sharing clock for the per-chunk load measurement.  The
// CTAs resident on one SM share its FP64 pipe, so a tile's wall duration
// depends on how many neighbours it had (heavy tiles early in the heaviest-
// first queue run under full contention, the tail runs nearly alone).  Each
// SM keeps V(t) = integral dt / n_active(t); a tile is charged V(end) -
// V(start), its fair share of the SM.  The shares of all tiles on an SM sum to
// the SM's busy time, independent of the queue position of the tile.
// Updated by one thread per CTA at tile begin/end under a per-SM spin lock.
struct SmShare {
  int lock, n;
  unsigned long long t_last;
  double v, pad;
};
__device__ SmShare g_sm_share[1024];
__device__ int g_share_min_n = 1;  // OD_SHARE_MIN_N: floor of the divisor (diagnostic)
// diagnostic event log of the share clock (OD_TILELOG): {time, V, n, tag, sm, delta}
struct ShareEvent {
  unsigned long long t;
  double v;
  int n, tag, sm, delta;
};
__device__ ShareEvent* g_share_log = nullptr;
__device__ unsigned int g_share_log_n = 0;
__device__ unsigned int g_share_log_cap = 0;

__device__ __noinline__ double sm_share_update(int delta, int tag) {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  SmShare* s = &g_sm_share[sm & 1023];
  while (atomicCAS(&s->lock, 0, 1) != 0) __nanosleep(20);
  __threadfence();
  volatile SmShare* vs = s;
  const unsigned long long now = globaltimer_ns();
  double v = vs->v;
  const int n = vs->n;
  if (n > 0 && now > vs->t_last) v += double(now - vs->t_last) / double(n < g_share_min_n ? g_share_min_n : n);
  vs->v = v;
  vs->t_last = now;
  vs->n = n + delta;
  if (g_share_log) {
    const unsigned i = atomicAdd(&g_share_log_n, 1u);
    if (i < g_share_log_cap) g_share_log[i] = ShareEvent{now, v, n, tag, int(sm), delta};
  }
  __threadfence();
  atomicExch(&s->lock, 0);
  return v;
}

// A fused tile's share-clock account in shared memory: the tile is charged
// only while it can work.  A tile whose physics is exhausted and which blocks
// on a neighbour (peer strip, or a same-GPU tile still finishing the previous
// step under cross-step overlap) pauses its account and leaves the SM's
// resident count, so idling for a neighbour is charged to nobody and the
// other tiles on the SM get the SM.
struct ShareAcct {
  double t0, acc;
};
__device__ __forceinline__ void share_begin(ShareAcct& a, int tag) {
  a.acc = 0.0;
  a.t0 = sm_share_update(1, tag);
}
__device__ __forceinline__ void share_pause(ShareAcct& a, int tag) {
  a.acc += sm_share_update(-1, tag) - a.t0;
}
__device__ __forceinline__ void share_resume(ShareAcct& a, int tag) {
  a.t0 = sm_share_update(1, tag);
}
__device__ __forceinline__ double share_end(ShareAcct& a, int tag) {
  return a.acc + (sm_share_update(-1, tag) - a.t0);
}

// Executed FP64 pipe instructions, the work measure that apportions a GPU's
// measured busy time among its chunks (TIMER): one physics trip is 2*n_inner+3
// (two FMAs per unit, the trip's y and eb), one Jacobi cell 8 (6 add, mul, fma).
__device__ __forceinline__ unsigned long long trip_ops(int n_inner) {
  return 2ull * (unsigned long long)n_inner + 3ull;
}
constexpr unsigned long long kJacobiOps = 8;

// chunk_ns rows hold (share ns, executed ops) per slot: add this thread's ops,
// one atomic per warp.  Every lane of the warp must call it.
__device__ __forceinline__ void charge_ops(unsigned long long* __restrict__ chunk_ns, int slot,
                                           unsigned long long ops) {
  for (int o = 16; o > 0; o >>= 1) ops += __shfl_down_sync(0xffffffffu, ops, o);
  if ((threadIdx.x & 31) == 0 && ops) atomicAdd(&chunk_ns[2 * slot + 1], ops);
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin (one thread) until every sender has published `stamp`; trap after
// timeout_ns so a dead peer fails the step loudly instead of hanging it.
__device__ __forceinline__ void wait_stamps(const unsigned long long* __restrict__ flags,
                                            const int32_t* __restrict__ senders, int32_t n,
                                            unsigned long long stamp, uint64_t timeout_ns) {
  for (int i = 0; i < n; ++i) {
    const unsigned long long* f = flags + senders[i];
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(f) < stamp) {
      if (globaltimer_ns() - t0 > timeout_ns) __trap();
      __nanosleep(64);
    }
  }
}

// Peer-halo dependency of one tile (persistent kernels, P2P halos): the
// senders' step flags to poll; n == 0 when the tile needs nothing remote or the
// strips are known to have landed.
constexpr int kPreroll = 256;  // physics units per pre-roll round (multiple of 16)

// P2P halos are published per face: the sender's pack stores the stamp into
// flags[fbase + 4 * vp + side] on the receiving GPU (vp: the receiving chunk,
// side: its face) once all fields of that strip have landed, so a tile waits
// only for the strips it reads, not for every strip of every sender.
struct HaloWait {
  const unsigned long long* flags;
  int32_t fbase;  // flags[fbase + 4 * vp + side]
  int32_t n;      // bit mask of the remote faces this tile reads (0: none)
  unsigned long long stamp;
  unsigned long long* wait_ns;  // longest blocking wait (diagnostic), may be null
  // cross-step overlap: neighbour tiles on this GPU that must have finished the
  // previous step (their U^t cells are this tile's halo)
  const unsigned* done;
  const int32_t* deps;
  int32_t ndeps;
  unsigned need;
};

__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ bool stamps_ready(const HaloWait& hw) {
  for (int d = 0; d < 4; ++d)
    if (((hw.n >> d) & 1) && ld_acquire_sys(hw.flags + hw.fbase + d) < hw.stamp) return false;
  for (int i = 0; i < hw.ndeps; ++i)
    if (ld_acquire_gpu_u32(hw.done + hw.deps[i]) < hw.need) return false;
  return true;
}

// spin (one thread) until stamps_ready; trap after timeout_ns
__device__ __forceinline__ void wait_ready(const HaloWait& hw, uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer_ns();
  while (!stamps_ready(hw)) {
    if (globaltimer_ns() - t0 > timeout_ns) __trap();
    __nanosleep(64);
  }
}

// Cross-step overlap of the step kernels (PDL): per-tile completion stamps and,
// per tile, the tiles of this GPU whose cells it reads as halo (itself first).
struct StepDeps {
  const int32_t* off;   // [ntiles + 1] CSR over canonical tile ids
  const int32_t* idx;
  const int32_t* joff;  // [njobs + 1] pack job -> tiles holding its face cells
  const int32_t* jidx;
  unsigned* done;       // [ntiles] steps completed per tile
  unsigned long long* end_ns;  // this step's last tile end (globaltimer), may be null
  unsigned step;        // steps completed before this one
  int32_t on;
  // host-facing steps: the CTA finishing the step's last tile writes the step's
  // per-chunk measurement row straight into mapped pinned host memory
  unsigned* tile_cnt;   // tiles of this step finished so far
  int32_t ntiles, res_words;
  unsigned long long* res_dst;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// the same with the shared address already converted (compile-time slot
// offsets then fold into the instruction's immediate)
__device__ __forceinline__ void cp_async8s(uint32_t s, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16s(uint32_t s, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// shared loads at a register + compile-time byte offset
template <int OFF>
__device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];\n" : "=d"(v.x), "=d"(v.y) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ double lds1(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];\n" : "=d"(v) : "r"(a), "n"(OFF));
  return v;
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// CTA-scope mbarrier in shared memory: arrive (release) and wait for a phase
// (acquire) are separate, so a thread can signal "my reads of the ring are done
// and my copies have landed" and then run physics while the others catch up.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  uint64_t state;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];\n"
               : "=l"(state)
               : "r"(smem_u32(b))
               : "memory");
  (void)state;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}

// f(b, a) of Fig. 1 / Fig. 4: mix a and b, then n micro-steps of the
// perturbed logistic map.  Every operation is a correctly rounded add/mul/fma.
__device__ __forceinline__ double column_f(double b, double a, int n) {
  const double hb = __dmul_rn(0.5, b);
  const double eb = __fma_rn(b, kEps, kEps);
  double y = __fma_rn(0.5, a, hb);
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const double u = __fma_rn(-y, y, y);
    y = __fma_rn(kR, u, eb);
  }
  return y;
}

// ---------------------------------------------------------------------------
// Jacobi.  Grid (tiles, F); block (TX, TY).  A CTA marches its TX x TY column
// tile through the nz levels of one field.  Plane k (tile + 1-cell halo) is
// staged in smem slot k % R by cp.async, S planes ahead of the compute.
// ---------------------------------------------------------------------------
template <int TX, int TY, int S, bool TIMED>
__global__ void __launch_bounds__(TX* TY)
    jacobi_step(const ChunkDev* __restrict__ chunks, const TileDev* __restrict__ tiles,
                int32_t nz, unsigned long long* __restrict__ chunk_ns) {
  constexpr int R = S + 2;
  __shared__ __align__(16) double ring[R][TY + 2][TX + 2];

  double t_start = 0;
  if (TIMED && threadIdx.x == 0 && threadIdx.y == 0) t_start = sm_share_update(1, share_tag(tiles[blockIdx.x]));

  const TileDev tile = tiles[blockIdx.x];
  const ChunkDev& c = chunks[tile.slot];
  const int f = blockIdx.y;
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int w = c.w, h = c.h, pitch = c.pitch;
  const int64_t ks = c.kstride;
  const int wv = min(TX, w - tile.tx0), hv = min(TY, h - tile.ty0);
  const int x = tile.tx0 + lx, y = tile.ty0 + ly;
  const bool act = lx < wv && ly < hv;
  const double* src = c.in + f * c.fstride;
  double* dst = c.out + f * c.fstride;

  // center element of this thread
  const double* pc = src + int64_t(y) * pitch + x;
  // x-halo duty (left by lane 0, right by lane TX-1) for rows inside the tile
  const double* phx = nullptr;
  int64_t hxk = 0;
  int hx_col = 0;
  if (ly < hv && (lx == 0 || lx == TX - 1)) {
    const bool left = lx == 0;
    const int xs = left ? tile.tx0 - 1 : tile.tx0 + wv;
    hx_col = left ? 0 : wv + 1;
    if (xs >= 0 && xs < w) {
      phx = src + int64_t(y) * pitch + xs;
      hxk = ks;
    } else {
      const FaceDev& fd = c.face[left ? kLeft : kRight];
      phx = fd.p + f * fd.fs + int64_t(y) * fd.es;
      hxk = fd.ks;
    }
  }
  // y-halo duty (top by row 0, bottom by row TY-1) for columns inside the tile
  const double* phy = nullptr;
  int64_t hyk = 0;
  int hy_row = 0;
  if (lx < wv && (ly == 0 || ly == TY - 1)) {
    const bool top = ly == 0;
    const int ys = top ? tile.ty0 - 1 : tile.ty0 + hv;
    hy_row = top ? 0 : hv + 1;
    if (ys >= 0 && ys < h) {
      phy = src + int64_t(ys) * pitch + x;
      hyk = ks;
    } else {
      const FaceDev& fd = c.face[top ? kTop : kBottom];
      phy = fd.p + f * fd.fs + int64_t(x) * fd.es;
      hyk = fd.ks;
    }
  }

  auto issue = [&](int k) {
    if (k < nz) {
      const int s = k % R;
      if (act) cp_async8(&ring[s][ly + 1][lx + 1], pc + k * ks);
      if (phx) cp_async8(&ring[s][ly + 1][hx_col], phx + k * hxk);
      if (phy) cp_async8(&ring[s][hy_row][lx + 1], phy + k * hyk);
    }
    cp_async_commit();
  };

#pragma unroll
  for (int k = 0; k < S; ++k) issue(k);

  for (int k = 0; k < nz; ++k) {
    cp_async_wait<S - 2>();  // planes <= k+1 have landed for this thread
    __syncthreads();         // ... and for every thread; slot of plane k-2 is free
    issue(k + S);
    if (act) {
      const int s0 = k % R;
      const double uc = ring[s0][ly + 1][lx + 1];
      const double xm = ring[s0][ly + 1][lx];
      const double xp = ring[s0][ly + 1][lx + 2];
      const double ym = ring[s0][ly][lx + 1];
      const double yp = ring[s0][ly + 2][lx + 1];
      const double zm = k > 0 ? ring[(k + R - 1) % R][ly + 1][lx + 1] : uc;
      const double zp = k + 1 < nz ? ring[(k + 1) % R][ly + 1][lx + 1] : uc;
      const double s =
          __dadd_rn(__dadd_rn(__dadd_rn(xm, xp), __dadd_rn(ym, yp)), __dadd_rn(zm, zp));
      const double v = __fma_rn(kW1, s, __dmul_rn(kW0, uc));
      __stcs(dst + int64_t(y) * pitch + x + k * ks, v);
    }
  }
  cp_async_wait<0>();

  if (TIMED) {
    charge_ops(chunk_ns, tile.slot, act ? kJacobiOps * (unsigned long long)nz : 0ull);
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0)
      atomicAdd(&chunk_ns[2 * tile.slot], (unsigned long long)llrint(sm_share_update(-1, share_tag(tile)) - t_start));
  }
}

// ---------------------------------------------------------------------------
// Physics.  Grid (tiles); block (TX, TY); one thread per column.  B is field 0
// of U^t (read-only this step, so the kernel is independent of jacobi_step).
// ---------------------------------------------------------------------------
// One column of the recurrence; returns its trip count (0 for threads outside
// the chunk).  A(l) = f(B(l), A(l-1)), l = t mod nz for t = 1..T.
__device__ __forceinline__ int physics_column(const ChunkDev& c, const TileDev& tile, int lx,
                                              int ly, const double* __restrict__ cfield,
                                              int32_t nx, int32_t ny, int32_t shift, int32_t nz,
                                              int32_t n_inner) {
  const int x = tile.tx0 + lx, y = tile.ty0 + ly;
  if (x >= c.w || y >= c.h) return 0;
  int row = c.y0 + y - shift;
  if (row < 0) row += ny;
  const double cm = __ldg(cfield + int64_t(row) * nx + c.x0 + x);
  int T = int(floor(__dmul_rn(double(nz), cm))) - 1;
  if (T < 0) T = 0;
  const int64_t ks = c.kstride;
  const double* B = c.in + int64_t(y) * c.pitch + x;  // field 0 of U^t
  double* A = c.a + int64_t(y) * c.pitch + x;
  double a = A[0];
  int ln = nz > 1 ? 1 : 0;
  double bn = T >= 1 ? B[ln * ks] : 0.0;
  for (int t = 1; t <= T; ++t) {
    const int l = ln;
    const double b = bn;
    ln = l + 1 == nz ? 0 : l + 1;
    if (t < T) bn = B[ln * ks];  // prefetch the next level
    a = column_f(b, a, n_inner);
    A[l * ks] = a;
  }
  return T;
}

// Physics.  Grid (tiles); block (TX, TY); one thread per column.  B is field 0
// of U^t (read-only this step, so the kernel is independent of jacobi_step).
template <int TX, int TY, bool TIMED, bool COUNT>
__global__ void __launch_bounds__(TX* TY)
    physics_step(const ChunkDev* __restrict__ chunks, const TileDev* __restrict__ tiles,
                 const double* __restrict__ cfield, int32_t nx, int32_t ny, int32_t shift,
                 int32_t nz, int32_t n_inner, unsigned long long* __restrict__ chunk_ns,
                 unsigned long long* __restrict__ trips) {
  double t_start = 0;
  if (TIMED && threadIdx.x == 0 && threadIdx.y == 0) t_start = sm_share_update(1, share_tag(tiles[blockIdx.x]));
  const TileDev tile = tiles[blockIdx.x];
  const int T = physics_column(chunks[tile.slot], tile, threadIdx.x, threadIdx.y, cfield, nx, ny,
                               shift, nz, n_inner);
  if (COUNT) {
    unsigned long long v = (unsigned long long)T;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&trips[tile.slot], v);
  }
  if (TIMED) {
    charge_ops(chunk_ns, tile.slot, (unsigned long long)(T > 0 ? T : 0) * trip_ops(n_inner));
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0)
      atomicAdd(&chunk_ns[2 * tile.slot], (unsigned long long)llrint(sm_share_update(-1, share_tag(tile)) - t_start));
  }
}

// ---------------------------------------------------------------------------
// Fused step.  On B200 a kernel that saturates the FP64 pipe starves every
// co-resident warp that needs that pipe (tools/overlap_probe.cu: a copy with 7
// FP64 ops/element drops from 4.0 TB/s to 0.8 TB/s next to an FP64-FMA kernel),
// so running the physics and the Jacobi as two concurrent kernels does not
// overlap them.  Here the SAME warps interleave both: after every Jacobi level
// step (one plane of one field) each thread advances its column recurrence by
// a fixed quota of work units, so the Jacobi's loads are in flight while the
// FP64 pipe runs the recurrence.  Results are bitwise identical to running
// jacobi_step and physics_step back to back (same operations, same order per
// value).  Grid (tiles); block (TX, TY).
// ---------------------------------------------------------------------------
struct ColumnState {
  const double* B;  // field 0 of U^t at this column
  double* A;
  int64_t ks;
  int T, t, i, l, nz, n_inner;
  double a, y, eb, bn;
};

__device__ __forceinline__ void physics_init(ColumnState& s, const ChunkDev& c, int x, int y,
                                             const double* __restrict__ cfield, int32_t nx,
                                             int32_t ny, int32_t shift, int32_t nz,
                                             int32_t n_inner) {
  int row = c.y0 + y - shift;
  if (row < 0) row += ny;
  OD_CHECK(row >= 0 && row < ny && c.x0 + x >= 0 && c.x0 + x < nx, "physics: load field index");
  const double cm = __ldg(cfield + int64_t(row) * nx + c.x0 + x);
  int T = int(floor(__dmul_rn(double(nz), cm))) - 1;
  s.T = T < 0 ? 0 : T;
  OD_CHECK(c.a + int64_t(y) * c.pitch + x + int64_t(nz - 1) * c.kstride < c.a + int64_t(nz) * c.kstride,
           "physics: A range");
  s.ks = c.kstride;
  s.B = c.in + int64_t(y) * c.pitch + x;
  s.A = c.a + int64_t(y) * c.pitch + x;
  s.nz = nz;
  s.n_inner = n_inner;
  s.t = 1;
  s.i = 0;
  s.l = nz > 1 ? 1 : 0;
  s.a = s.A[0];
  s.y = 0.0;
  s.eb = 0.0;
  s.bn = s.T >= 1 ? s.B[s.l * s.ks] : 0.0;
}

// Advance by `budget` work units: a trip is 1 setup unit + n_inner micro-steps.
// Callers pass budgets that are multiples of 8 (or "everything") so the common
// case -- the budget ends inside the current trip -- is a fully unrolled loop.
__device__ __forceinline__ void physics_advance(ColumnState& s, int budget) {
  if (s.i > 0 && budget <= s.n_inner - s.i) {  // (no overflow for "everything" budgets)
    double y = s.y;
    const double eb = s.eb;
    for (int j = 0; j < budget; j += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double u = __fma_rn(-y, y, y);
        y = __fma_rn(kR, u, eb);
      }
    }
    s.y = y;
    s.i += budget;
    return;
  }
  while (budget > 0 && s.t <= s.T) {
    if (s.i == 0) {
      const double b = s.bn;
      const double hb = __dmul_rn(0.5, b);
      s.eb = __fma_rn(b, kEps, kEps);
      s.y = __fma_rn(0.5, s.a, hb);
      s.i = 1;
      --budget;
      const int ln = s.l + 1 == s.nz ? 0 : s.l + 1;
      if (s.t < s.T) s.bn = s.B[ln * s.ks];
    }
    const int m = min(budget, s.n_inner + 1 - s.i);
    double y = s.y;
    const double eb = s.eb;
#pragma unroll 16
    for (int j = 0; j < m; ++j) {
      const double u = __fma_rn(-y, y, y);
      y = __fma_rn(kR, u, eb);
    }
    s.y = y;
    s.i += m;
    budget -= m;
    if (s.i == s.n_inner + 1) {
      s.a = y;
      s.A[s.l * s.ks] = y;
      s.l = s.l + 1 == s.nz ? 0 : s.l + 1;
      ++s.t;
      s.i = 0;
    }
  }
}

// Two columns with the same trip count advance in lockstep (equal budgets from
// the same quota), so their trip boundaries coincide: handle both chains
// together, interleaved, across the boundary -- the same operations per
// chain as physics_advance, in the same order.
__device__ __forceinline__ void physics_advance_pair(ColumnState& s0, ColumnState& s1,
                                                     int budget) {
  while (budget > 0 && s0.t <= s0.T) {
    if (s0.i == 0) {
      const double b0 = s0.bn, b1 = s1.bn;
      const double hb0 = __dmul_rn(0.5, b0), hb1 = __dmul_rn(0.5, b1);
      s0.eb = __fma_rn(b0, kEps, kEps);
      s1.eb = __fma_rn(b1, kEps, kEps);
      s0.y = __fma_rn(0.5, s0.a, hb0);
      s1.y = __fma_rn(0.5, s1.a, hb1);
      s0.i = s1.i = 1;
      --budget;
      const int ln = s0.l + 1 == s0.nz ? 0 : s0.l + 1;
      if (s0.t < s0.T) {
        s0.bn = s0.B[ln * s0.ks];
        s1.bn = s1.B[ln * s1.ks];
      }
    }
    const int m = min(budget, s0.n_inner + 1 - s0.i);
    double y0 = s0.y, y1 = s1.y;
    const double e0 = s0.eb, e1 = s1.eb;
#pragma unroll 16
    for (int j = 0; j < m; ++j) {
      const double u0 = __fma_rn(-y0, y0, y0);
      const double u1 = __fma_rn(-y1, y1, y1);
      y0 = __fma_rn(kR, u0, e0);
      y1 = __fma_rn(kR, u1, e1);
    }
    s0.y = y0;
    s1.y = y1;
    s0.i += m;
    s1.i += m;
    budget -= m;
    if (s0.i == s0.n_inner + 1) {
      s0.a = y0;
      s1.a = y1;
      s0.A[s0.l * s0.ks] = y0;
      s1.A[s1.l * s1.ks] = y1;
      s0.l = s1.l = s0.l + 1 == s0.nz ? 0 : s0.l + 1;
      ++s0.t;
      ++s1.t;
      s0.i = s1.i = 0;
    }
  }
}

// Calls of physics_advance(s, budget) that stay inside the current trip.
__device__ __forceinline__ int fast_calls(const ColumnState& s, int budget) {
  return (s.i > 0 && budget > 0 && s.t <= s.T) ? (s.n_inner - s.i) / budget : 0;
}

// ---------------------------------------------------------------------------
// Fused tile kernels.  A tile is tw x th columns of one chunk: tw in {8, 16, 32,
// 64} is chosen per chunk width on the host (tile_shape in od_runtime.cu), a
// thread owns two adjacent columns of one row, so a warp covers 64 / tw rows of
// tw / 2 threads and the four row-warps of a CTA cover th = 256 / tw rows.
// Narrow chunks (cfg3's 32, cfg1's 16, cfg2's 8 columns) thus fill every lane
// of a warp instead of leaving lanes 16..31 without a column.  The ring plane
// is (th + 2) x (tw + 4) doubles ([pad][left halo][tw][right halo][pad]): at
// most 408 doubles for every shape.
// ---------------------------------------------------------------------------
constexpr int kRingSlots = 8;
constexpr int kPlaneMax = 416;  // >= (th + 2) * (tw + 4) over the four shapes; 128-byte multiple (TMA)
constexpr int kRowWarps = 4;

struct TileGeom {
  int tw, th, pw;  // tile width, height, ring row pitch
  int lx, ly;      // this thread's column pair and row inside the tile
};

// row warp `wr` (0..3) and lane of this thread
__device__ __forceinline__ TileGeom tile_geom(const TileDev& t, int wr, int lane) {
  TileGeom g;
  g.tw = t.tw;
  g.th = t.th;
  g.pw = t.tw + 4;
  const int lg = t.lg;  // log2(tw / 2): threads per row = 1 << lg
  g.lx = lane & ((1 << lg) - 1);
  g.ly = wr * (32 >> lg) + (lane >> lg);
  return g;
}

// One tile, all fields and levels: the Jacobi of every (field, level) plane
// through a cp.async plane ring (two levels per mbarrier phase) interleaved in
// the same warps with the two physics recurrences of each thread.  Uniform
// plane strides (fs == nz * ks holds for chunk buffers, neighbour faces and
// packed receive faces alike, so every walker is p += ks) and a countdown that
// keeps the two chains on the branch-free interleaved loop between trip
// boundaries.  FULL: the tile lies inside the chunk (compile-time two cells
// per thread, no partial-tile predicates).  Same arithmetic as every path.
template <int S, bool TIMED, bool FULL, int R = kRingSlots>
__device__ __forceinline__ void tile_step(double* __restrict__ ring, const TileDev tile,
                                          const ChunkDev* __restrict__ chunks, int32_t nz,
                                          int32_t F, const double* __restrict__ cfield,
                                          int32_t nx, int32_t ny, int32_t shift, int32_t n_inner,
                                          unsigned long long* __restrict__ chunk_ns,
                                          const HaloWait hw) {
  static_assert((R & (R - 1)) == 0, "ring slots: power of two");
  static_assert(S + 2 <= R && S >= 3, "prefetch depth");
  __shared__ ShareAcct s_acct;
  if (TIMED && threadIdx.x == 0 && threadIdx.y == 0) share_begin(s_acct, share_tag(tile));

  const ChunkDev& c = chunks[tile.slot];
  const TileGeom g = tile_geom(tile, threadIdx.y, threadIdx.x);
  const int PW = g.pw, PLANE = (g.th + 2) * PW;
  const int lx = g.lx, ly = g.ly;
  const int w = c.w, h = c.h, pitch = c.pitch;
  const int64_t ks = c.kstride;
  const int wv = FULL ? g.tw : min(g.tw, w - tile.tx0);
  const int hv = FULL ? g.th : min(g.th, h - tile.ty0);
  const int x = tile.tx0 + 2 * lx, y = tile.ty0 + ly;
  // cells of this thread's pair inside the chunk (compile-time 2 for full tiles)
  const int pair = FULL ? 2 : max(0, min(2, wv - 2 * lx));
  const int ncell = FULL ? 2 : (ly < hv ? pair : 0);
  const int64_t own = int64_t(y) * pitch + x;
  const int tpr = g.tw >> 1;

  const double* pc = c.in + own;
  const double* px = nullptr;
  const double* py = nullptr;
  int64_t xstep = 0, ystep = 0;
  int ox = 0, oy = 0, ny_cells = 0;
  const double* const in_hi = c.in + int64_t(F) * c.fstride;
  const double *xlo = c.in, *xhi = in_hi, *ylo = c.in, *yhi = in_hi;  // walker allocations
  if (ly < hv && (lx == 0 || lx == tpr - 1)) {
    // x-halo duty: the row's first thread loads the left, its last the right
    // halo cell (a one-thread row, tw = 2, never occurs: tw >= 8)
    const bool left = lx == 0;
    const int xs = left ? tile.tx0 - 1 : tile.tx0 + wv;
    ox = (ly + 1) * PW + (left ? 1 : wv + 2);
    if (xs >= 0 && xs < w) {
      px = c.in + int64_t(y) * pitch + xs;
      xstep = ks;
    } else {
      const FaceDev& fd = c.face[left ? kLeft : kRight];
      px = fd.p + int64_t(y) * fd.es;
      xstep = fd.ks;
      xlo = fd.lo;
      xhi = fd.hi;
    }
  }
  if (pair > 0 && (ly == 0 || ly == g.th - 1)) {
    const bool top = ly == 0;
    const int ys = top ? tile.ty0 - 1 : tile.ty0 + hv;
    oy = (top ? 0 : hv + 1) * PW + 2 + 2 * lx;
    ny_cells = pair;
    if (ys >= 0 && ys < h) {
      py = c.in + int64_t(ys) * pitch + x;
      ystep = ks;
    } else {
      const FaceDev& fd = c.face[top ? kTop : kBottom];
      py = fd.p + int64_t(x) * fd.es;
      ystep = fd.ks;
      ylo = fd.lo;
      yhi = fd.hi;
    }
  }
  const int oc = (ly + 1) * PW + 2 + 2 * lx;
  const int levels = F * nz;
#ifdef OD_CHECKED
  {
    const int64_t span = int64_t(levels - 1) * ks;
    if (ncell > 0) {
      OD_CHECK(od_in(pc, c.in, in_hi) && od_in(pc + span + ncell - 1, c.in, in_hi),
               "tile: U^t read range");
      OD_CHECK(od_in(c.out + own, c.out, c.out + int64_t(F) * c.fstride) &&
                   od_in(c.out + own + span + ncell - 1, c.out, c.out + int64_t(F) * c.fstride),
               "tile: U^{t+1} write range");
      OD_CHECK(oc >= PW && oc + 2 <= (g.th + 1) * PW && oc + 2 <= kPlaneMax, "tile: ring offset");
    }
    if (px) {
      OD_CHECK(od_in(px, xlo, xhi) && od_in(px + int64_t(levels - 1) * xstep, xlo, xhi),
               "tile: x-halo read range");
      OD_CHECK(ox >= 0 && ox < kPlaneMax, "tile: x-halo ring offset");
    }
    if (py) {
      OD_CHECK(od_in(py, ylo, yhi) && od_in(py + int64_t(levels - 1) * ystep + ny_cells - 1, ylo, yhi),
               "tile: y-halo read range");
      OD_CHECK(oy >= 0 && oy + ny_cells <= kPlaneMax, "tile: y-halo ring offset");
    }
  }
#endif

  auto issue = [&](int L) {
    if (L < levels) {
      double* slot = ring + (L & (R - 1)) * kPlaneMax;
      if (ncell == 2) cp_async16(slot + oc, pc);
      else if (ncell == 1) cp_async8(slot + oc, pc);
      if (px) cp_async8(slot + ox, px);
      if (ny_cells == 2) cp_async16(slot + oy, py);
      else if (ny_cells == 1) cp_async8(slot + oy, py);
      pc += ks;
      px += xstep;
      py += ystep;
    }
    cp_async_commit();
  };
  // the same without the bound test (callers know L < levels; full tiles)
  auto issue_full = [&](int L) {
    double* slot = ring + (L & (R - 1)) * kPlaneMax;
    cp_async16(slot + oc, pc);
    if (px) cp_async8(slot + ox, px);
    if (ny_cells == 2) cp_async16(slot + oy, py);
    pc += ks;
    px += xstep;
    py += ystep;
    cp_async_commit();
  };

  // slot-constant copies: SLOT known at compile time (the 8-level unrolled loop)
  const uint32_t sh_c = static_cast<uint32_t>(__cvta_generic_to_shared(ring + oc));
  const uint32_t sh_x = static_cast<uint32_t>(__cvta_generic_to_shared(ring + ox));
  const uint32_t sh_y = static_cast<uint32_t>(__cvta_generic_to_shared(ring + oy));
  const uint32_t sh_m = sh_c - uint32_t(PW) * 8u, sh_p = sh_c + uint32_t(PW) * 8u;
  // the plane stride re-read from shared memory through a thread-dependent
  // address, so it lives in a vector register: the walkers' 64-bit steps use
  // it directly instead of copying it out of a uniform register at each use
  __shared__ int64_t s_ks[1];
  if (threadIdx.x == 0 && threadIdx.y == 0) s_ks[0] = ks;
  int64_t ksv = ks;  // re-read after the ring barrier's __syncthreads below
  auto issue_slot = [&](auto slot) {
    constexpr uint32_t off = uint32_t(decltype(slot)::value) * kPlaneMax * 8u;
    cp_async16s(sh_c + off, pc);
    if (px) cp_async8s(sh_x + off, px);
    if (ny_cells == 2) cp_async16s(sh_y + off, py);
    pc += ksv;
    px += xstep;
    py += ystep;
    cp_async_commit();
  };

  ColumnState s0, s1;
  int q0 = 0, q1 = 0;
  if (ncell >= 1) {
    physics_init(s0, c, x, y, cfield, nx, ny, shift, nz, n_inner);
    q0 = int((int64_t(s0.T) * (n_inner + 1) + levels - 1) / levels);
    q0 = (q0 + 15) & ~15;
  }
  if (ncell == 2) {
    physics_init(s1, c, x + 1, y, cfield, nx, ny, shift, nz, n_inner);
    q1 = int((int64_t(s1.T) * (n_inner + 1) + levels - 1) / levels);
    q1 = (q1 + 15) & ~15;
  }
  int fast = 0;  // interleaved iterations left before a trip boundary
  auto physics = [&](int b0, int b1) {
    if (fast > 0) {
      double y0 = s0.y, y1 = s1.y;
      const double e0 = s0.eb, e1 = s1.eb;
      // b0 is a multiple of 32 (quota rounded to 16, two levels per call)
      for (int j = 0; j < b0; j += 32) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const double u0 = __fma_rn(-y0, y0, y0);
          const double u1 = __fma_rn(-y1, y1, y1);
          y0 = __fma_rn(kR, u0, e0);
          y1 = __fma_rn(kR, u1, e1);
        }
      }
      s0.y = y0;
      s1.y = y1;
      s0.i += b0;
      s1.i += b0;
      --fast;
      return;
    }
    if (ncell == 2 && b0 == b1 && s0.T == s1.T) {
      physics_advance_pair(s0, s1, b0);  // lockstep columns: keep both chains interleaved
      fast = min(fast_calls(s0, b0), fast_calls(s1, b1));
      return;
    }
    if (ncell >= 1) physics_advance(s0, b0);
    if (ncell == 2) {
      physics_advance(s1, b1);
      if (b0 == b1) fast = min(fast_calls(s0, b0), fast_calls(s1, b1));
    }
  };

  // one level of one field for this thread's cells (plane in slot L & 7)
  double zm0 = 0.0, zm1 = 0.0;
  double* pout = c.out + own;
  const double* rc = ring + oc;
  auto level = [&](int L, int k) {
    const double* pl = rc + (L & (R - 1)) * kPlaneMax;
    if (ncell == 2) {
      const double2 uc = *reinterpret_cast<const double2*>(pl);
      const double xl = pl[-1], xr = pl[2];
      const double2 ym = *reinterpret_cast<const double2*>(pl - PW);
      const double2 yp = *reinterpret_cast<const double2*>(pl + PW);
      double2 zu = uc;
      if (k + 1 < nz) zu = *reinterpret_cast<const double2*>(rc + ((L + 1) & (R - 1)) * kPlaneMax);
      const double zd0 = k > 0 ? zm0 : uc.x, zd1 = k > 0 ? zm1 : uc.y;
      const double sa = __dadd_rn(__dadd_rn(__dadd_rn(xl, uc.y), __dadd_rn(ym.x, yp.x)),
                                  __dadd_rn(zd0, zu.x));
      const double sb = __dadd_rn(__dadd_rn(__dadd_rn(uc.x, xr), __dadd_rn(ym.y, yp.y)),
                                  __dadd_rn(zd1, zu.y));
      double2 o;
      o.x = __fma_rn(kW1, sa, __dmul_rn(kW0, uc.x));
      o.y = __fma_rn(kW1, sb, __dmul_rn(kW0, uc.y));
      __stcs(reinterpret_cast<double2*>(pout), o);
      zm0 = uc.x;
      zm1 = uc.y;
    } else if (ncell == 1) {
      const double uc = pl[0];
      const double zu = k + 1 < nz ? rc[((L + 1) & (R - 1)) * kPlaneMax] : uc;
      const double zd = k > 0 ? zm0 : uc;
      const double sum = __dadd_rn(__dadd_rn(__dadd_rn(pl[-1], pl[1]), __dadd_rn(pl[-PW], pl[PW])),
                                   __dadd_rn(zd, zu));
      __stcs(pout, __fma_rn(kW1, sum, __dmul_rn(kW0, uc)));
      zm0 = uc;
    }
    pout += ks;
  };
  (void)PLANE;
  // full-tile level with its k position known: FIRST (k == 0: no level below),
  // LAST (k == nz - 1: no level above), neither -- no per-level predicates
  auto level_k = [&](int L, auto first, auto last) {
    const double* pl = rc + (L & (R - 1)) * kPlaneMax;
    const double2 uc = *reinterpret_cast<const double2*>(pl);
    const double xl = pl[-1], xr = pl[2];
    const double2 ym = *reinterpret_cast<const double2*>(pl - PW);
    const double2 yp = *reinterpret_cast<const double2*>(pl + PW);
    double2 zu = uc;
    if (!decltype(last)::value)
      zu = *reinterpret_cast<const double2*>(rc + ((L + 1) & (R - 1)) * kPlaneMax);
    const double zd0 = decltype(first)::value ? uc.x : zm0;
    const double zd1 = decltype(first)::value ? uc.y : zm1;
    const double sa = __dadd_rn(__dadd_rn(__dadd_rn(xl, uc.y), __dadd_rn(ym.x, yp.x)),
                                __dadd_rn(zd0, zu.x));
    const double sb = __dadd_rn(__dadd_rn(__dadd_rn(uc.x, xr), __dadd_rn(ym.y, yp.y)),
                                __dadd_rn(zd1, zu.y));
    double2 o;
    o.x = __fma_rn(kW1, sa, __dmul_rn(kW0, uc.x));
    o.y = __fma_rn(kW1, sb, __dmul_rn(kW0, uc.y));
    __stcs(reinterpret_cast<double2*>(pout), o);
    zm0 = uc.x;
    zm1 = uc.y;
    pout += ks;
  };

  // the same with the slot (and the next level's) known at compile time
  // the same with the slot known at compile time: every plane read is a
  // register + immediate shared load; the level's centre plane comes in as
  // `uc` (the level below read it as its upper neighbour) and its upper
  // neighbour goes out as the next level's centre
  auto level_s = [&](auto slot, auto first, auto last, double2 uc) -> double2 {
    constexpr int sl = decltype(slot)::value;
    constexpr int off = sl * kPlaneMax * 8;
    constexpr int offn = ((sl + 1) & (R - 1)) * kPlaneMax * 8;
    const double xl = lds1<off - 8>(sh_c), xr = lds1<off + 16>(sh_c);
    const double2 ym = lds2<off>(sh_m);
    const double2 yp = lds2<off>(sh_p);
    double2 zu = uc;
    if (!decltype(last)::value) zu = lds2<offn>(sh_c);
    const double zd0 = decltype(first)::value ? uc.x : zm0;
    const double zd1 = decltype(first)::value ? uc.y : zm1;
    const double sa = __dadd_rn(__dadd_rn(__dadd_rn(xl, uc.y), __dadd_rn(ym.x, yp.x)),
                                __dadd_rn(zd0, zu.x));
    const double sb = __dadd_rn(__dadd_rn(__dadd_rn(uc.x, xr), __dadd_rn(ym.y, yp.y)),
                                __dadd_rn(zd1, zu.y));
    double2 o;
    o.x = __fma_rn(kW1, sa, __dmul_rn(kW0, uc.x));
    o.y = __fma_rn(kW1, sb, __dmul_rn(kW0, uc.y));
    __stcs(reinterpret_cast<double2*>(pout), o);
    zm0 = uc.x;
    zm1 = uc.y;
    pout += ksv;
    return zu;
  };

  if (hw.n > 0 || hw.ndeps > 0) {
    // The tile reads strips a peer GPU stores into this GPU's receive buffer
    // during this step, or cells of same-GPU tiles still finishing the previous
    // step.  Until they are there, run the tile's physics (which reads only
    // this tile's own U^t): the wait costs the SM nothing while the physics
    // lasts, so such tiles can sit anywhere in the heaviest-first queue.
    const int64_t need = int64_t(max(ncell >= 1 ? s0.T : 0, ncell == 2 ? s1.T : 0)) * (n_inner + 1);
    int64_t done = 0;
    bool lead_ready = false;
    for (;;) {
      const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
      if (lead) {
        if (done >= need) {
          // physics exhausted before the strips came: block (traps on a dead
          // peer) with the tile's account paused (idling is charged to nobody)
          if (TIMED) share_pause(s_acct, share_tag(tile));
          const uint64_t w0 = globaltimer_ns();
          wait_ready(hw, 20ull * 1000 * 1000 * 1000);
          if (hw.wait_ns) atomicMax(hw.wait_ns, (unsigned long long)(globaltimer_ns() - w0));
          if (TIMED) share_resume(s_acct, share_tag(tile));
          lead_ready = true;
        } else {
          lead_ready = stamps_ready(hw);
        }
      }
      if (__syncthreads_or(lead && lead_ready)) break;
      physics(kPreroll, kPreroll);
      done += kPreroll;
    }
    fast = 0;  // the level loop's budgets differ from the pre-roll's
  }

  // ring hand-off: an mbarrier phase per level pair.  A thread arrives once its
  // reads of the pair's planes are done and its copies for the next pair have
  // landed, then runs its physics quota while the other warps catch up; the
  // next pair starts (and refills the slots just read) when the phase is done.
  __shared__ uint64_t s_ring_bar;
  const bool bar_lead = threadIdx.x == 0 && threadIdx.y == 0;
  if (bar_lead) mbar_init(&s_ring_bar, blockDim.x * blockDim.y);
  __syncthreads();
  ksv = s_ks[threadIdx.y >> 3];  // (index 0: blockDim.y <= 8)

#pragma unroll
  for (int L = 0; L < S; ++L) issue(L);
  cp_async_wait<S - 3>();  // planes <= 2 landed for this thread
  mbar_arrive(&s_ring_bar);

  uint32_t parity = 0;
  int k = 0, L = 0;
  if (FULL && R == 8 && (nz & 7) == 0) {
    // nz a multiple of 8: the level loop unrolled over the 8 ring slots, so
    // every plane address is a register plus an immediate (no per-level slot
    // arithmetic); the first and last pair of a field are peeled as below
    using T_ = std::true_type;
    using F_ = std::false_type;
    double2 ucn = make_double2(0.0, 0.0);  // the next level's centre plane
    // IN_RANGE: every copy of the 8-level block is below `levels`
    auto pair = [&](auto P, auto first, auto last, auto in_range) {
      constexpr int p = decltype(P)::value;
      mbar_wait(&s_ring_bar, parity);
      parity ^= 1;
      if (decltype(in_range)::value) {
        issue_slot(std::integral_constant<int, (2 * p + S) & 7>{});
        issue_slot(std::integral_constant<int, (2 * p + S + 1) & 7>{});
      } else {
        issue(L + S);
        issue(L + S + 1);
      }
      if (decltype(first)::value) ucn = lds2<2 * p * kPlaneMax * 8>(sh_c);
      ucn = level_s(std::integral_constant<int, 2 * p>{}, first, F_{}, ucn);
      ucn = level_s(std::integral_constant<int, 2 * p + 1>{}, F_{}, last, ucn);
      cp_async_wait<S - 3>();
      od_jitter(4u + unsigned(L));
      mbar_arrive(&s_ring_bar);
      physics(2 * q0, 2 * q1);
      L += 2;
    };
    using P0 = std::integral_constant<int, 0>;
    using P1 = std::integral_constant<int, 1>;
    using P2 = std::integral_constant<int, 2>;
    using P3 = std::integral_constant<int, 3>;
    for (int f = 0; f < F; ++f) {
      for (int kk = 0; kk < nz; kk += 8) {
        auto block = [&](auto in_range) {
          if (kk == 0) pair(P0{}, T_{}, F_{}, in_range);
          else pair(P0{}, F_{}, F_{}, in_range);
          pair(P1{}, F_{}, F_{}, in_range);
          pair(P2{}, F_{}, F_{}, in_range);
          if (kk == nz - 8) pair(P3{}, F_{}, T_{}, in_range);
          else pair(P3{}, F_{}, F_{}, in_range);
        };
        if (L + S + 8 <= levels) block(T_{});
        else block(F_{});
      }
    }
  } else if (FULL && (nz & 1) == 0 && nz >= 4) {
    // even nz: a level pair never straddles two fields; the first and last
    // pair of a field are peeled so the levels carry no k tests, and the
    // copies skip their bound test until the last S planes
    using T_ = std::true_type;
    using F_ = std::false_type;
    const int tail = levels - S - 2;  // pairs with L <= tail copy planes < levels
    for (int f = 0; f < F; ++f) {
      for (int kk = 0; kk < nz; kk += 2, L += 2) {
        mbar_wait(&s_ring_bar, parity);
        parity ^= 1;
        if (L <= tail) {
          issue_full(L + S);
          issue_full(L + S + 1);
        } else {
          issue(L + S);
          issue(L + S + 1);
        }
        if (kk == 0) {
          level_k(L, T_{}, F_{});
          level_k(L + 1, F_{}, F_{});
        } else if (kk == nz - 2) {
          level_k(L, F_{}, F_{});
          level_k(L + 1, F_{}, T_{});
        } else {
          level_k(L, F_{}, F_{});
          level_k(L + 1, F_{}, F_{});
        }
        cp_async_wait<S - 3>();  // this thread's planes <= L+4 landed
        od_jitter(4u + unsigned(L));
        mbar_arrive(&s_ring_bar);
        physics(2 * q0, 2 * q1);
      }
    }
  }
  for (; L + 1 < levels; L += 2) {
    mbar_wait(&s_ring_bar, parity);  // everyone: planes <= L+2 landed, planes L-2, L-1 read
    parity ^= 1;
    issue(L + S);
    issue(L + S + 1);
    level(L, k);
    if (++k == nz) k = 0;
    level(L + 1, k);
    if (++k == nz) k = 0;
    cp_async_wait<S - 3>();  // this thread's planes <= L+4 landed
    od_jitter(4u + unsigned(L));
    mbar_arrive(&s_ring_bar);
    physics(2 * q0, 2 * q1);
  }
  if (L < levels) {
    mbar_wait(&s_ring_bar, parity);
    level(L, k);
  }
  cp_async_wait<0>();
  __syncthreads();
  if (bar_lead) mbar_inval(&s_ring_bar);
  if (ncell >= 1) physics_advance(s0, 0x7fffffff);
  if (ncell == 2) physics_advance(s1, 0x7fffffff);

  if (TIMED) {
    unsigned long long ops = (unsigned long long)ncell * nz * F * kJacobiOps;
    if (ncell >= 1) ops += (unsigned long long)s0.T * trip_ops(n_inner);
    if (ncell == 2) ops += (unsigned long long)s1.T * trip_ops(n_inner);
    charge_ops(chunk_ns, tile.slot, ops);
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0)
      atomicAdd(&chunk_ns[2 * tile.slot], (unsigned long long)llrint(share_end(s_acct, share_tag(tile))));
  }
}

// Partial tiles (chunk edges narrower or shorter than the tile) take an
// out-of-line path so their predicates do not cost registers in the common
// full-tile code.
template <int S, bool TIMED, int R = kRingSlots>
__device__ __noinline__ void tile_step_partial(double* __restrict__ ring, const TileDev tile,
                                               const ChunkDev* __restrict__ chunks, int32_t nz,
                                               int32_t F, const double* __restrict__ cfield,
                                               int32_t nx, int32_t ny, int32_t shift,
                                               int32_t n_inner,
                                               unsigned long long* __restrict__ chunk_ns,
                                               const HaloWait hw) {
  tile_step<S, TIMED, false, R>(ring, tile, chunks, nz, F, cfield, nx, ny, shift, n_inner,
                                chunk_ns, hw);
}

// ---------------------------------------------------------------------------
// TMA-staged full tile (mode 4/5 interleaved kernel, tiles that lie inside
// their chunk).  Same tile shape, Jacobi arithmetic and physics interleave as
// tile_step, but each (field, level) plane of the tile lands in shared memory
// through the tensor memory accelerator: one elected thread issues, per
// plane, a tw x th box of the chunk's own U^t plus the two halo rows (from
// the chunk itself, the neighbour chunk's map, or the received strip's map),
// all completing on the plane slot's "full" mbarrier with expect-tx; the
// threads owning a row's first/last column pair copy the two x-halo cells
// (8 B each, not a TMA box) with cp.async and arrive on the same barrier
// (noinc).  Slot layout (doubles, 128-byte aligned regions):
//   [top row: tw (>= 16)] [tile: th x tw] [bottom row: tw (>= 16)] [x-halo: th x 2]
// The ring hand-off (slots refilled only after every thread has read them)
// is tile_step's mbarrier phase per level pair.
// ---------------------------------------------------------------------------
constexpr int kTmaSlot = kPlaneMax;  // doubles per slot (>= 392, every shape's TMA layout)

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensormap_acquire(const void* tmap) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(tmap) : "memory");
}

template <int S, bool TIMED>
__device__ __forceinline__ void tile_step_tma(double* __restrict__ ring, const TileDev tile,
                                              const ChunkDev* __restrict__ chunks, int32_t nz,
                                              int32_t F, const double* __restrict__ cfield,
                                              int32_t nx, int32_t ny, int32_t shift,
                                              int32_t n_inner,
                                              unsigned long long* __restrict__ chunk_ns,
                                              const HaloWait hw) {
  constexpr int R = kRingSlots;
  static_assert(S + 2 <= R && S >= 3, "prefetch depth");
  __shared__ ShareAcct s_acct;
  if (TIMED && threadIdx.x == 0 && threadIdx.y == 0) share_begin(s_acct, share_tag(tile));

  const ChunkDev& c = chunks[tile.slot];
  const TileGeom g = tile_geom(tile, threadIdx.y, threadIdx.x);
  const int tw = g.tw, th = g.th;
  const int lx = g.lx, ly = g.ly;
  const int pitch = c.pitch;
  const int64_t ks = c.kstride;
  const int x = tile.tx0 + 2 * lx, y = tile.ty0 + ly;
  const int64_t own = int64_t(y) * pitch + x;
  const int tpr = tw >> 1;
  const int levels = F * nz;

  // slot layout
  const int row_len = tw < 16 ? 16 : tw;
  const int o_top = 0, o_main = row_len, o_bot = row_len + th * tw, o_xh = o_bot + row_len;
  const int oc = o_main + ly * tw + 2 * lx;
  const int o_ym = ly == 0 ? o_top + 2 * lx : oc - tw;
  const int o_yp = ly == th - 1 ? o_bot + 2 * lx : oc + tw;
  const int o_xl = lx == 0 ? o_xh + 2 * ly : oc - 1;
  const int o_xr = lx == tpr - 1 ? o_xh + 2 * ly + 1 : oc + 2;

  // x-halo duty: the row's first and last thread copy one cell each per plane
  const double* px = nullptr;
  int64_t xstep = 0;
  int oxh = 0;
  if (lx == 0 || lx == tpr - 1) {
    const bool left = lx == 0;
    const int xs = left ? tile.tx0 - 1 : tile.tx0 + tw;
    oxh = o_xh + 2 * ly + (left ? 0 : 1);
    if (xs >= 0 && xs < c.w) {
      px = c.in + int64_t(y) * pitch + xs;
      xstep = ks;
    } else {
      const FaceDev& fd = c.face[left ? kLeft : kRight];
      px = fd.p + int64_t(y) * fd.es;
      xstep = fd.ks;
    }
  }
  // halo rows: sources resolved once (uniform over the CTA)
  const FaceDev& ft = c.face[kTop];
  const FaceDev& fb = c.face[kBottom];
  const bool top_in = tile.ty0 > 0, bot_in = tile.ty0 + th < c.h;
  const void* tm_top = top_in ? c.tm_row : ft.tm;
  const void* tm_bot = bot_in ? c.tm_row : fb.tm;
  const int top_y = top_in ? tile.ty0 - 1 : ft.trow;
  const int bot_y = bot_in ? tile.ty0 + th : fb.trow;
  const bool top_2d = !top_in && ft.tkind == 1, bot_2d = !bot_in && fb.tkind == 1;
  const uint32_t tx_bytes = uint32_t((th + 2) * tw) * 8u;

  __shared__ __align__(8) uint64_t s_full[R];
  __shared__ uint64_t s_ring_bar;
  const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
  if (lead) {
    for (int i = 0; i < R; ++i) mbar_init(&s_full[i], 1 + 2 * th);
    mbar_init(&s_ring_bar, blockDim.x * blockDim.y);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x == 0) {  // the issuing lanes
    tensormap_acquire(c.tm_main);
    tensormap_acquire(c.tm_row);
    tensormap_acquire(tm_top);
    tensormap_acquire(tm_bot);
  }

  // the issuing thread rotates over the four warps' first lanes, so no warp
  // carries the TMA issue of every plane
  const int wid = threadIdx.y;
  auto issue = [&](int L) {
    if (L >= levels) return;
    double* slot = ring + (L & (R - 1)) * kTmaSlot;
    uint64_t* full = &s_full[L & (R - 1)];
    if (threadIdx.x == 0 && wid == ((L >> 1) & (kRowWarps - 1))) {
      mbar_expect_tx(full, tx_bytes);
      tma_load_3d(slot + o_main, c.tm_main, tile.tx0, tile.ty0, L, full);
      if (top_2d) tma_load_2d(slot + o_top, tm_top, tile.tx0, L, full);
      else tma_load_3d(slot + o_top, tm_top, tile.tx0, top_y, L, full);
      if (bot_2d) tma_load_2d(slot + o_bot, tm_bot, tile.tx0, L, full);
      else tma_load_3d(slot + o_bot, tm_bot, tile.tx0, bot_y, L, full);
    }
    if (px) {
      cp_async8(slot + oxh, px);
      cp_async_mbar_arrive_noinc(full);
      px += xstep;
    }
  };
  auto wait_plane = [&](int L) {
    if (L < levels) mbar_wait(&s_full[L & (R - 1)], uint32_t((L / R) & 1));
  };

  ColumnState s0, s1;
  physics_init(s0, c, x, y, cfield, nx, ny, shift, nz, n_inner);
  physics_init(s1, c, x + 1, y, cfield, nx, ny, shift, nz, n_inner);
  int q0 = int((int64_t(s0.T) * (n_inner + 1) + levels - 1) / levels);
  q0 = (q0 + 15) & ~15;
  int q1 = int((int64_t(s1.T) * (n_inner + 1) + levels - 1) / levels);
  q1 = (q1 + 15) & ~15;
  int fast = 0;
  auto physics = [&](int b0, int b1) {
    if (fast > 0) {
      double y0 = s0.y, y1 = s1.y;
      const double e0 = s0.eb, e1 = s1.eb;
      for (int j = 0; j < b0; j += 32) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const double u0 = __fma_rn(-y0, y0, y0);
          const double u1 = __fma_rn(-y1, y1, y1);
          y0 = __fma_rn(kR, u0, e0);
          y1 = __fma_rn(kR, u1, e1);
        }
      }
      s0.y = y0;
      s1.y = y1;
      s0.i += b0;
      s1.i += b0;
      --fast;
      return;
    }
    if (b0 == b1 && s0.T == s1.T) {
      physics_advance_pair(s0, s1, b0);
      fast = min(fast_calls(s0, b0), fast_calls(s1, b1));
      return;
    }
    physics_advance(s0, b0);
    physics_advance(s1, b1);
    if (b0 == b1) fast = min(fast_calls(s0, b0), fast_calls(s1, b1));
  };

  double zm0 = 0.0, zm1 = 0.0;
  double* pout = c.out + own;
  auto level = [&](int L, int k) {
    const double* pl = ring + (L & (R - 1)) * kTmaSlot;
    const double2 uc = *reinterpret_cast<const double2*>(pl + oc);
    const double xl = pl[o_xl], xr = pl[o_xr];
    const double2 ym = *reinterpret_cast<const double2*>(pl + o_ym);
    const double2 yp = *reinterpret_cast<const double2*>(pl + o_yp);
    double2 zu = uc;
    if (k + 1 < nz)
      zu = *reinterpret_cast<const double2*>(ring + ((L + 1) & (R - 1)) * kTmaSlot + oc);
    const double zd0 = k > 0 ? zm0 : uc.x, zd1 = k > 0 ? zm1 : uc.y;
    const double sa = __dadd_rn(__dadd_rn(__dadd_rn(xl, uc.y), __dadd_rn(ym.x, yp.x)),
                                __dadd_rn(zd0, zu.x));
    const double sb = __dadd_rn(__dadd_rn(__dadd_rn(uc.x, xr), __dadd_rn(ym.y, yp.y)),
                                __dadd_rn(zd1, zu.y));
    double2 o;
    o.x = __fma_rn(kW1, sa, __dmul_rn(kW0, uc.x));
    o.y = __fma_rn(kW1, sb, __dmul_rn(kW0, uc.y));
    __stcs(reinterpret_cast<double2*>(pout), o);
    zm0 = uc.x;
    zm1 = uc.y;
    pout += ks;
  };

  if (hw.n > 0 || hw.ndeps > 0) {
    // pre-roll the physics until the remote strips / neighbour tiles are there
    const int64_t need = int64_t(max(s0.T, s1.T)) * (n_inner + 1);
    int64_t done = 0;
    bool lead_ready = false;
    for (;;) {
      if (lead) {
        if (done >= need) {
          if (TIMED) share_pause(s_acct, share_tag(tile));
          const uint64_t w0 = globaltimer_ns();
          wait_ready(hw, 20ull * 1000 * 1000 * 1000);
          if (hw.wait_ns) atomicMax(hw.wait_ns, (unsigned long long)(globaltimer_ns() - w0));
          if (TIMED) share_resume(s_acct, share_tag(tile));
          lead_ready = true;
        } else {
          lead_ready = stamps_ready(hw);
        }
      }
      if (__syncthreads_or(lead && lead_ready)) break;
      physics(kPreroll, kPreroll);
      done += kPreroll;
    }
    fast = 0;
  }
  // U^t and the received strips were written through the generic proxy (the
  // previous step's tiles, the peers' pack CTAs) and acquired through the step
  // stamps / halo flags; order those writes before this tile's TMA reads
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;\n" ::: "memory");
  __syncthreads();  // barriers initialised (and the pre-roll's stamps acquired) before any TMA

#pragma unroll
  for (int L = 0; L < S; ++L) issue(L);
  mbar_arrive(&s_ring_bar);

  uint32_t parity = 0;
  int k = 0, L = 0;
  for (; L + 1 < levels; L += 2) {
    mbar_wait(&s_ring_bar, parity);  // everyone has read planes <= L-1: their slots are free
    parity ^= 1;
    issue(L + S);
    issue(L + S + 1);
    if (L == 0) wait_plane(L);  // (later: plane L was waited for as L+2 one phase ago)
    wait_plane(L + 1);
    wait_plane(L + 2);
    level(L, k);
    if (++k == nz) k = 0;
    level(L + 1, k);
    if (++k == nz) k = 0;
    od_jitter(4u + unsigned(L));
    mbar_arrive(&s_ring_bar);
    physics(2 * q0, 2 * q1);
  }
  if (L < levels) {
    mbar_wait(&s_ring_bar, parity);
    wait_plane(L);
    level(L, k);
  }
  cp_async_wait<0>();
  __syncthreads();
  if (lead) {
    for (int i = 0; i < R; ++i) mbar_inval(&s_full[i]);
    mbar_inval(&s_ring_bar);
  }
  physics_advance(s0, 0x7fffffff);
  physics_advance(s1, 0x7fffffff);

  if (TIMED) {
    unsigned long long ops = 2ull * nz * F * kJacobiOps;
    ops += (unsigned long long)s0.T * trip_ops(n_inner);
    ops += (unsigned long long)s1.T * trip_ops(n_inner);
    charge_ops(chunk_ns, tile.slot, ops);
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0)
      atomicAdd(&chunk_ns[2 * tile.slot], (unsigned long long)llrint(share_end(s_acct, share_tag(tile))));
  }
}

__device__ __forceinline__ bool tile_full(const TileDev& t, const ChunkDev& c) {
  return t.tx0 + t.tw <= c.w && t.ty0 + t.th <= c.h;
}

// Halo pack fused into the step kernel (P2P halos): the first `ctas` CTAs
// store this step's boundary strips straight into the peers' receive buffers
// over NVLink, one (face, field) unit at a time; the other CTAs start on tiles
// at once, so the NVLink transfer overlaps the compute.  The CTA that
// completes the last unit publishes the step to the peers (same protocol as
// pack_faces_p2p).
struct PackArgs {
  const PackJob* jobs;
  int32_t njobs, ctas;
  double* const* peer_base;
  int64_t half_elems;
  int32_t par, n_notify, my_rank, first;  // first: lowest blockIdx that packs
  unsigned int* counters;  // [next unit, units done], zeroed before the launch
  unsigned int* jcnt;      // per job: fields packed this step, zeroed before the launch
  unsigned long long* const* peer_flags;
  const int32_t* notify;
};

__device__ __noinline__ void pack_units(const PackArgs pk, const ChunkDev* __restrict__ chunks,
                                        int32_t nz, int32_t F, unsigned long long stamp,
                                        const StepDeps sd) {
  __shared__ int s_unit;
  const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nthr = blockDim.x * blockDim.y;
  const int total = pk.njobs * F;
  for (;;) {
    if (lead) s_unit = int(atomicAdd(&pk.counters[0], 1u));
    __syncthreads();
    const int u = s_unit;
    __syncthreads();
    if (u >= total) break;
    if (sd.on) {
      // the face cells are U^t of this GPU's edge tiles: wait for their step
      if (lead) {
        const int jb = u / F;
        const uint64_t t0 = globaltimer_ns();
        for (int q = sd.joff[jb]; q < sd.joff[jb + 1]; ++q)
          while (ld_acquire_gpu_u32(sd.done + sd.jidx[q]) < sd.step) {
            if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) __trap();
            __nanosleep(32);
          }
      }
      __syncthreads();
    }
    const PackJob j = pk.jobs[u / F];
    const int f = u - (u / F) * F;
    const ChunkDev& c = chunks[j.slot];
    const double* base = c.in + f * c.fstride;
    int64_t off = 0, es = 1;
    switch (j.side) {
      case kLeft: off = 0; es = c.pitch; break;
      case kRight: off = c.w - 1; es = c.pitch; break;
      case kTop: off = 0; es = 1; break;
      default: off = int64_t(c.h - 1) * c.pitch; es = 1; break;
    }
    double* out = pk.peer_base[j.peer] + int64_t(pk.par) * pk.half_elems + j.rdst +
                  int64_t(f) * nz * j.lenp;
    // (level, position) flattened; 8 independent loads in flight per thread
    const int n = nz * j.len;
    OD_CHECK(j.rdst >= 0 && j.rdst + (int64_t(f) + 1) * nz * j.lenp <= pk.half_elems,
             "pack: peer strip range");
    OD_CHECK(off + int64_t(nz - 1) * c.kstride + int64_t(j.len - 1) * es < c.fstride,
             "pack: face read range");
    constexpr int U = 8;
    for (int i0 = tid; i0 < n; i0 += U * nthr) {
      double v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int i = i0 + q * nthr;
        if (i < n) {
          const int k = i / j.len, e = i - k * j.len;
          v[q] = __ldcs(base + off + k * c.kstride + int64_t(e) * es);
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int i = i0 + q * nthr;
        if (i < n) {
          const int k = i / j.len, e = i - k * j.len;
          out[int64_t(k) * j.lenp + e] = v[q];
        }
      }
    }
    __threadfence_system();
    __syncthreads();
    od_jitter(3u);
    // the last field of a strip publishes that strip to its reader
    if (lead && atomicAdd(&pk.jcnt[u / F], 1u) == unsigned(F - 1)) {
      __threadfence_system();
      st_release_sys(pk.peer_flags[j.peer] + j.rflag, stamp);
    }
    if (lead && atomicAdd(&pk.counters[1], 1u) == unsigned(total - 1)) {
      __threadfence_system();
      for (int i = 0; i < pk.n_notify; ++i)
        st_release_sys(pk.peer_flags[pk.notify[i]] + pk.my_rank, stamp);
    }
  }
}

// Remote faces of chunk c that tile t touches (bit d: face d), i.e. the strips it reads.
__device__ __forceinline__ int tile_remote_faces(const TileDev& t, const ChunkDev& c) {
  int m = 0;
  if (t.tx0 == 0) m |= 1 << kLeft;
  if (t.tx0 + t.tw >= c.w) m |= 1 << kRight;
  if (t.ty0 == 0) m |= 1 << kTop;
  if (t.ty0 + t.th >= c.h) m |= 1 << kBottom;
  return m & c.rmask;
}

// Cross-step overlap, tile side: block on the tile's own previous step (its
// columns' A and U^t), then hand the same-GPU neighbour tiles to tile_step's
// pre-roll poll.
__device__ __forceinline__ void tile_deps(const StepDeps& sd, int self, HaloWait& hw) {
  if (!sd.on) return;
  od_jitter(1u);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_gpu_u32(sd.done + self) < sd.step) {
      if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) __trap();
      __nanosleep(32);
    }
  }
  __syncthreads();
  hw.done = sd.done;
  hw.deps = sd.idx + sd.off[self] + 1;
  hw.ndeps = sd.off[self + 1] - sd.off[self] - 1;
  hw.need = sd.step;
}

// Publish the tile's step; the CTA that finishes the step's last tile copies
// the step's per-chunk measurement row into mapped pinned host memory.
__device__ __forceinline__ void tile_publish(const StepDeps& sd, int self,
                                             const unsigned long long* __restrict__ chunk_ns) {
  if (!sd.on) return;
  __syncthreads();  // every thread's U^{t+1} stores issued
  __shared__ int s_last;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    od_jitter(2u);
    __threadfence();
    st_release_gpu_u32(sd.done + self, sd.step + 1);
    if (sd.end_ns) atomicMax(sd.end_ns, (unsigned long long)globaltimer_ns());
    s_last = sd.res_dst ? atomicAdd(sd.tile_cnt, 1u) == unsigned(sd.ntiles - 1) : 0;
  }
  if (sd.res_dst) {
    __syncthreads();
    if (s_last) {
      __threadfence();  // every tile's shares are in
      const int tid = threadIdx.y * blockDim.x + threadIdx.x;
      for (int i = tid; i < sd.res_words; i += blockDim.x * blockDim.y)
        sd.res_dst[i] = __ldcg(chunk_ns + i);
      __threadfence_system();
    }
  }
}

// Mode 4 (and mode 5 from one wave of tiles up): one CTA (4 row-warps) per
// tile over the heaviest-first tile list.  The block scheduler starts CTAs in
// index order as earlier ones retire, and the warp scheduler favours older
// warps, so tiles are served roughly first-come-first-served.  With P2P halos
// the first pk.ctas CTAs only pack this step's boundary strips into the peers'
// buffers and exit; with sd.on the grid is launched with programmatic
// dependent launch behind the previous step's (cross-step overlap).
template <int S, bool TIMED, int MINB, int R = kRingSlots>
__global__ void __launch_bounds__(32 * kRowWarps, MINB)
    column_step_grid(const ChunkDev* __restrict__ chunks, const TileDev* __restrict__ tiles,
                     int32_t nz, int32_t F, const double* __restrict__ cfield, int32_t nx,
                     int32_t ny, int32_t shift, int32_t n_inner,
                     unsigned long long* __restrict__ chunk_ns,
                     const unsigned long long* __restrict__ halo_flags, int32_t face_base,
                     unsigned long long stamp, unsigned long long* __restrict__ wait_ns,
                     const PackArgs pk, const StepDeps sd) {
  // rings deeper than 8 slots exceed the 48 KB static limit: dynamic smem
  __shared__ __align__(128) double ring_s[R <= 8 ? R * kPlaneMax : 2];
  extern __shared__ __align__(128) double ring_d[];
  double* const ring = R <= 8 ? ring_s : ring_d;
  // cross-step overlap: let the next step's grid launch as soon as every CTA of
  // this one has started; its tiles wait on per-tile stamps, not on this grid
  if (sd.on) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (int(blockIdx.x) < pk.ctas) {
    if (pk.njobs > 0) pack_units(pk, chunks, nz, F, stamp, sd);
    return;
  }
  const TileDev t = tiles[blockIdx.x - pk.ctas];
  const ChunkDev& c = chunks[t.slot];
  const int self = t.pad >> 1;
  HaloWait hw{halo_flags, face_base + 4 * c.vp, (t.pad & 1) ? tile_remote_faces(t, c) : 0,
              stamp, wait_ns, nullptr, nullptr, 0, 0};
  tile_deps(sd, self, hw);
  if (tile_full(t, c) && c.tm_main && R == kRingSlots)
    tile_step_tma<S, TIMED>(ring, t, chunks, nz, F, cfield, nx, ny, shift, n_inner, chunk_ns, hw);
  else if (tile_full(t, c))
    tile_step<S, TIMED, true, R>(ring, t, chunks, nz, F, cfield, nx, ny, shift, n_inner, chunk_ns,
                                 hw);
  else
    tile_step_partial<S, TIMED, R>(ring, t, chunks, nz, F, cfield, nx, ny, shift, n_inner,
                                   chunk_ns, hw);
  tile_publish(sd, self, chunk_ns);
}

// Warp-specialised tile (mode 7; mode 5 when a GPU holds less than one wave of
// tiles): the same tile shapes, ring and Jacobi code as tile_step, but 8 warps:
// warps 0..3 run only the physics of their rows' column pairs (chains back to
// back, no ring, no barrier) while warps 4..7 stream the Jacobi planes of the
// same rows.  A tile lasts max(physics, Jacobi) instead of their sum, which is
// what counts when the GPU holds few tiles (latency-bound sizes).
template <int S, bool TIMED, bool FULL>
__device__ __forceinline__ void tile_step_ws(double* __restrict__ ring, const TileDev tile,
                                             const ChunkDev* __restrict__ chunks, int32_t nz,
                                             int32_t F, const double* __restrict__ cfield,
                                             int32_t nx, int32_t ny, int32_t shift,
                                             int32_t n_inner,
                                             unsigned long long* __restrict__ chunk_ns,
                                             const HaloWait hw) {
  constexpr int R = kRingSlots;
  static_assert(S + 2 <= R && S >= 3, "prefetch depth");
  __shared__ ShareAcct s_acct;
  __shared__ int s_phys_left;  // physics warps still running (TIMED: pause when idle)
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    s_phys_left = kRowWarps;
    if (TIMED) share_begin(s_acct, share_tag(tile));
  }

  const ChunkDev& c = chunks[tile.slot];
  // warp roles: threadIdx.y < 4 physics, >= 4 Jacobi, both over row warp y % 4
  const bool phys = threadIdx.y < kRowWarps;
  const TileGeom g = tile_geom(tile, threadIdx.y % kRowWarps, threadIdx.x);
  const int PW = g.pw;
  const int lx = g.lx, ly = g.ly;
  const int w = c.w, h = c.h, pitch = c.pitch;
  const int64_t ks = c.kstride;
  const int wv = FULL ? g.tw : min(g.tw, w - tile.tx0);
  const int hv = FULL ? g.th : min(g.th, h - tile.ty0);
  const int x = tile.tx0 + 2 * lx, y = tile.ty0 + ly;
  const int pair = FULL ? 2 : max(0, min(2, wv - 2 * lx));
  const int ncell = FULL ? 2 : (ly < hv ? pair : 0);
  const int64_t own = int64_t(y) * pitch + x;
  const int tpr = g.tw >> 1;

  const double* pc = c.in + own;
  const double* px = nullptr;
  const double* py = nullptr;
  int64_t xstep = 0, ystep = 0;
  int ox = 0, oy = 0, ny_cells = 0;
  const double* const in_hi = c.in + int64_t(F) * c.fstride;
  const double *xlo = c.in, *xhi = in_hi, *ylo = c.in, *yhi = in_hi;  // walker allocations
  if (!phys && ly < hv && (lx == 0 || lx == tpr - 1)) {
    const bool left = lx == 0;
    const int xs = left ? tile.tx0 - 1 : tile.tx0 + wv;
    ox = (ly + 1) * PW + (left ? 1 : wv + 2);
    if (xs >= 0 && xs < w) {
      px = c.in + int64_t(y) * pitch + xs;
      xstep = ks;
    } else {
      const FaceDev& fd = c.face[left ? kLeft : kRight];
      px = fd.p + int64_t(y) * fd.es;
      xstep = fd.ks;
      xlo = fd.lo;
      xhi = fd.hi;
    }
  }
  if (!phys && pair > 0 && (ly == 0 || ly == g.th - 1)) {
    const bool top = ly == 0;
    const int ys = top ? tile.ty0 - 1 : tile.ty0 + hv;
    oy = (top ? 0 : hv + 1) * PW + 2 + 2 * lx;
    ny_cells = pair;
    if (ys >= 0 && ys < h) {
      py = c.in + int64_t(ys) * pitch + x;
      ystep = ks;
    } else {
      const FaceDev& fd = c.face[top ? kTop : kBottom];
      py = fd.p + int64_t(x) * fd.es;
      ystep = fd.ks;
      ylo = fd.lo;
      yhi = fd.hi;
    }
  }
  const int oc = (ly + 1) * PW + 2 + 2 * lx;
  const int levels = F * nz;
#ifdef OD_CHECKED
  {
    const int64_t span = int64_t(levels - 1) * ks;
    if (ncell > 0) {
      OD_CHECK(od_in(pc, c.in, in_hi) && od_in(pc + span + ncell - 1, c.in, in_hi),
               "tile: U^t read range");
      OD_CHECK(od_in(c.out + own, c.out, c.out + int64_t(F) * c.fstride) &&
                   od_in(c.out + own + span + ncell - 1, c.out, c.out + int64_t(F) * c.fstride),
               "tile: U^{t+1} write range");
      OD_CHECK(oc >= PW && oc + 2 <= (g.th + 1) * PW && oc + 2 <= kPlaneMax, "tile: ring offset");
    }
    if (px) {
      OD_CHECK(od_in(px, xlo, xhi) && od_in(px + int64_t(levels - 1) * xstep, xlo, xhi),
               "tile: x-halo read range");
      OD_CHECK(ox >= 0 && ox < kPlaneMax, "tile: x-halo ring offset");
    }
    if (py) {
      OD_CHECK(od_in(py, ylo, yhi) && od_in(py + int64_t(levels - 1) * ystep + ny_cells - 1, ylo, yhi),
               "tile: y-halo read range");
      OD_CHECK(oy >= 0 && oy + ny_cells <= kPlaneMax, "tile: y-halo ring offset");
    }
  }
#endif

  auto issue = [&](int L) {
    if (L < levels) {
      double* slot = ring + (L & (R - 1)) * kPlaneMax;
      if (ncell == 2) cp_async16(slot + oc, pc);
      else if (ncell == 1) cp_async8(slot + oc, pc);
      if (px) cp_async8(slot + ox, px);
      if (ny_cells == 2) cp_async16(slot + oy, py);
      else if (ny_cells == 1) cp_async8(slot + oy, py);
      pc += ks;
      px += xstep;
      py += ystep;
    }
    cp_async_commit();
  };
  // full tiles: slot-constant copies and levels, as in tile_step
  const uint32_t sh_c = static_cast<uint32_t>(__cvta_generic_to_shared(ring + oc));
  const uint32_t sh_x = static_cast<uint32_t>(__cvta_generic_to_shared(ring + ox));
  const uint32_t sh_y = static_cast<uint32_t>(__cvta_generic_to_shared(ring + oy));
  const uint32_t sh_m = sh_c - uint32_t(PW) * 8u, sh_p = sh_c + uint32_t(PW) * 8u;
  auto issue_slot = [&](auto slot) {
    constexpr uint32_t off = uint32_t(decltype(slot)::value) * kPlaneMax * 8u;
    cp_async16s(sh_c + off, pc);
    if (px) cp_async8s(sh_x + off, px);
    if (ny_cells == 2) cp_async16s(sh_y + off, py);
    pc += ks;
    px += xstep;
    py += ystep;
    cp_async_commit();
  };

  ColumnState s0, s1;
  if (phys && ncell >= 1) physics_init(s0, c, x, y, cfield, nx, ny, shift, nz, n_inner);
  if (phys && ncell == 2) physics_init(s1, c, x + 1, y, cfield, nx, ny, shift, nz, n_inner);

  double zm0 = 0.0, zm1 = 0.0;
  double* pout = c.out + own;
  const double* rc = ring + oc;
  auto level = [&](int L, int k) {
    const double* pl = rc + (L & (R - 1)) * kPlaneMax;
    if (ncell == 2) {
      const double2 uc = *reinterpret_cast<const double2*>(pl);
      const double xl = pl[-1], xr = pl[2];
      const double2 ym = *reinterpret_cast<const double2*>(pl - PW);
      const double2 yp = *reinterpret_cast<const double2*>(pl + PW);
      double2 zu = uc;
      if (k + 1 < nz) zu = *reinterpret_cast<const double2*>(rc + ((L + 1) & (R - 1)) * kPlaneMax);
      const double zd0 = k > 0 ? zm0 : uc.x, zd1 = k > 0 ? zm1 : uc.y;
      const double sa = __dadd_rn(__dadd_rn(__dadd_rn(xl, uc.y), __dadd_rn(ym.x, yp.x)),
                                  __dadd_rn(zd0, zu.x));
      const double sb = __dadd_rn(__dadd_rn(__dadd_rn(uc.x, xr), __dadd_rn(ym.y, yp.y)),
                                  __dadd_rn(zd1, zu.y));
      double2 o;
      o.x = __fma_rn(kW1, sa, __dmul_rn(kW0, uc.x));
      o.y = __fma_rn(kW1, sb, __dmul_rn(kW0, uc.y));
      __stcs(reinterpret_cast<double2*>(pout), o);
      zm0 = uc.x;
      zm1 = uc.y;
    } else if (ncell == 1) {
      const double uc = pl[0];
      const double zu = k + 1 < nz ? rc[((L + 1) & (R - 1)) * kPlaneMax] : uc;
      const double zd = k > 0 ? zm0 : uc;
      const double sum = __dadd_rn(__dadd_rn(__dadd_rn(pl[-1], pl[1]), __dadd_rn(pl[-PW], pl[PW])),
                                   __dadd_rn(zd, zu));
      __stcs(pout, __fma_rn(kW1, sum, __dmul_rn(kW0, uc)));
      zm0 = uc;
    }
    pout += ks;
  };
  auto level_s = [&](auto slot, auto first, auto last, double2 uc) -> double2 {
    constexpr int sl = decltype(slot)::value;
    constexpr int off = sl * kPlaneMax * 8;
    constexpr int offn = ((sl + 1) & (R - 1)) * kPlaneMax * 8;
    const double xl = lds1<off - 8>(sh_c), xr = lds1<off + 16>(sh_c);
    const double2 ym = lds2<off>(sh_m);
    const double2 yp = lds2<off>(sh_p);
    double2 zu = uc;
    if (!decltype(last)::value) zu = lds2<offn>(sh_c);
    const double zd0 = decltype(first)::value ? uc.x : zm0;
    const double zd1 = decltype(first)::value ? uc.y : zm1;
    const double sa = __dadd_rn(__dadd_rn(__dadd_rn(xl, uc.y), __dadd_rn(ym.x, yp.x)),
                                __dadd_rn(zd0, zu.x));
    const double sb = __dadd_rn(__dadd_rn(__dadd_rn(uc.x, xr), __dadd_rn(ym.y, yp.y)),
                                __dadd_rn(zd1, zu.y));
    double2 o;
    o.x = __fma_rn(kW1, sa, __dmul_rn(kW0, uc.x));
    o.y = __fma_rn(kW1, sb, __dmul_rn(kW0, uc.y));
    __stcs(reinterpret_cast<double2*>(pout), o);
    zm0 = uc.x;
    zm1 = uc.y;
    pout += ks;
    return zu;
  };

  __shared__ uint64_t s_ring_bar;
  const bool bar_lead = threadIdx.x == 0 && threadIdx.y == kRowWarps;  // first Jacobi thread
  if (bar_lead) mbar_init(&s_ring_bar, 32 * kRowWarps);
  __syncthreads();
  if (phys) {
    // physics warps: both chains to the end, nothing else
    if (ncell == 2 && s0.T == s1.T) {
      physics_advance_pair(s0, s1, 0x7fffffff);
    } else {
      if (ncell >= 1) physics_advance(s0, 0x7fffffff);
      if (ncell == 2) physics_advance(s1, 0x7fffffff);
    }
    __syncwarp();
    if (threadIdx.x == 0) atomicSub(&s_phys_left, 1);
  } else {
    // Jacobi warps: wait for remote strips / neighbour tiles, then stream the ring
    if (hw.n > 0 || hw.ndeps > 0) {
      if (bar_lead) {
        // wait while the physics warps work; once they are done and the
        // neighbours still are not, the tile idles: pause its account
        const uint64_t w0 = globaltimer_ns();
        bool paused = false;
        while (!stamps_ready(hw)) {
          if (TIMED && !paused && *(volatile int*)&s_phys_left == 0) {
            share_pause(s_acct, share_tag(tile));
            paused = true;
          }
          if (globaltimer_ns() - w0 > 20ull * 1000 * 1000 * 1000) __trap();
          __nanosleep(64);
        }
        if (TIMED && paused) share_resume(s_acct, share_tag(tile));
        if (hw.wait_ns) atomicMax(hw.wait_ns, (unsigned long long)(globaltimer_ns() - w0));
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kRowWarps) : "memory");
    }
#pragma unroll
    for (int L = 0; L < S; ++L) issue(L);
    cp_async_wait<S - 3>();
    mbar_arrive(&s_ring_bar);
    uint32_t parity = 0;
    int k = 0, L = 0;
    if (FULL && (nz & 7) == 0) {
      // the level loop unrolled over the 8 ring slots (see tile_step)
      using T_ = std::true_type;
      using F_ = std::false_type;
      double2 ucn = make_double2(0.0, 0.0);
      auto pair = [&](auto P, auto first, auto last, auto in_range) {
        constexpr int p = decltype(P)::value;
        mbar_wait(&s_ring_bar, parity);
        parity ^= 1;
        if (decltype(in_range)::value) {
          issue_slot(std::integral_constant<int, (2 * p + S) & 7>{});
          issue_slot(std::integral_constant<int, (2 * p + S + 1) & 7>{});
        } else {
          issue(L + S);
          issue(L + S + 1);
        }
        if (decltype(first)::value) ucn = lds2<2 * p * kPlaneMax * 8>(sh_c);
        ucn = level_s(std::integral_constant<int, 2 * p>{}, first, F_{}, ucn);
        ucn = level_s(std::integral_constant<int, 2 * p + 1>{}, F_{}, last, ucn);
        cp_async_wait<S - 3>();
        od_jitter(4u + unsigned(L));
        mbar_arrive(&s_ring_bar);
        L += 2;
      };
      using P0 = std::integral_constant<int, 0>;
      using P1 = std::integral_constant<int, 1>;
      using P2 = std::integral_constant<int, 2>;
      using P3 = std::integral_constant<int, 3>;
      for (int f = 0; f < F; ++f) {
        for (int kk = 0; kk < nz; kk += 8) {
          auto block = [&](auto in_range) {
            if (kk == 0) pair(P0{}, T_{}, F_{}, in_range);
            else pair(P0{}, F_{}, F_{}, in_range);
            pair(P1{}, F_{}, F_{}, in_range);
            pair(P2{}, F_{}, F_{}, in_range);
            if (kk == nz - 8) pair(P3{}, F_{}, T_{}, in_range);
            else pair(P3{}, F_{}, F_{}, in_range);
          };
          if (L + S + 8 <= levels) block(T_{});
          else block(F_{});
        }
      }
    }
    for (; L + 1 < levels; L += 2) {
      mbar_wait(&s_ring_bar, parity);
      parity ^= 1;
      issue(L + S);
      issue(L + S + 1);
      level(L, k);
      if (++k == nz) k = 0;
      level(L + 1, k);
      if (++k == nz) k = 0;
      cp_async_wait<S - 3>();
      od_jitter(4u + unsigned(L));
      mbar_arrive(&s_ring_bar);
    }
    if (L < levels) {
      mbar_wait(&s_ring_bar, parity);
      level(L, k);
    }
    cp_async_wait<0>();
  }
  __syncthreads();
  if (bar_lead) mbar_inval(&s_ring_bar);

  if (TIMED) {
    unsigned long long ops = 0;
    if (phys) {
      if (ncell >= 1) ops += (unsigned long long)s0.T * trip_ops(n_inner);
      if (ncell == 2) ops += (unsigned long long)s1.T * trip_ops(n_inner);
    } else {
      ops = (unsigned long long)ncell * nz * F * kJacobiOps;
    }
    charge_ops(chunk_ns, tile.slot, ops);
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0)
      atomicAdd(&chunk_ns[2 * tile.slot], (unsigned long long)llrint(share_end(s_acct, share_tag(tile))));
  }
}

template <int S, bool TIMED>
__device__ __noinline__ void tile_step_ws_partial(double* __restrict__ ring, const TileDev tile,
                                                  const ChunkDev* __restrict__ chunks, int32_t nz,
                                                  int32_t F, const double* __restrict__ cfield,
                                                  int32_t nx, int32_t ny, int32_t shift,
                                                  int32_t n_inner,
                                                  unsigned long long* __restrict__ chunk_ns,
                                                  const HaloWait hw) {
  tile_step_ws<S, TIMED, false>(ring, tile, chunks, nz, F, cfield, nx, ny, shift, n_inner,
                                chunk_ns, hw);
}

template <int S, bool TIMED, int MINB>
__global__ void __launch_bounds__(64 * kRowWarps, MINB)
    column_step_ws(const ChunkDev* __restrict__ chunks, const TileDev* __restrict__ tiles,
                   int32_t nz, int32_t F, const double* __restrict__ cfield, int32_t nx,
                   int32_t ny, int32_t shift, int32_t n_inner,
                   unsigned long long* __restrict__ chunk_ns,
                   const unsigned long long* __restrict__ halo_flags, int32_t face_base,
                   unsigned long long stamp, unsigned long long* __restrict__ wait_ns,
                   const PackArgs pk, const StepDeps sd) {
  __shared__ __align__(16) double ring[kRingSlots * kPlaneMax];
  if (sd.on) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (int(blockIdx.x) < pk.ctas) {
    if (pk.njobs > 0) pack_units(pk, chunks, nz, F, stamp, sd);
    return;
  }
  const TileDev t = tiles[blockIdx.x - pk.ctas];
  const ChunkDev& c = chunks[t.slot];
  const int self = t.pad >> 1;
  HaloWait hw{halo_flags, face_base + 4 * c.vp, (t.pad & 1) ? tile_remote_faces(t, c) : 0,
              stamp, wait_ns, nullptr, nullptr, 0, 0};
  tile_deps(sd, self, hw);
  if (tile_full(t, c))
    tile_step_ws<S, TIMED, true>(ring, t, chunks, nz, F, cfield, nx, ny, shift, n_inner, chunk_ns,
                                 hw);
  else
    tile_step_ws_partial<S, TIMED>(ring, t, chunks, nz, F, cfield, nx, ny, shift, n_inner,
                                   chunk_ns, hw);
  tile_publish(sd, self, chunk_ns);
}

// ---------------------------------------------------------------------------
// Face packing: grid (jobs, F); the strip of one field, all levels.
// Send layout per face: [f][k][e].
// ---------------------------------------------------------------------------
__global__ void pack_faces(const ChunkDev* __restrict__ chunks, const PackJob* __restrict__ jobs,
                           double* __restrict__ sendbuf, int32_t nz) {
  const PackJob j = jobs[blockIdx.x];
  const ChunkDev& c = chunks[j.slot];
  const int f = blockIdx.y;
  const double* base = c.in + f * c.fstride;
  int64_t off = 0, es = 1;
  switch (j.side) {
    case kLeft: off = 0; es = c.pitch; break;
    case kRight: off = c.w - 1; es = c.pitch; break;
    case kTop: off = 0; es = 1; break;
    default: off = int64_t(c.h - 1) * c.pitch; es = 1; break;
  }
  double* out = sendbuf + j.dst + int64_t(f) * nz * j.lenp;
  const int64_t n = int64_t(nz) * j.len;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t k = i / j.len, e = i - k * j.len;
    out[k * j.lenp + e] = base[off + k * c.kstride + e * es];
  }
}

// ---------------------------------------------------------------------------
// Halo exchange over NVLink peer memory: the pack kernel stores the boundary
// strips straight into the receive buffers of the neighbouring GPUs (CUDA IPC
// mappings), then the last CTA publishes the step number in each receiver's
// flag array (release, system scope).  The receiver's wait_halo acquires the
// flags before its step kernel reads the strips.  Receive buffers are double
// buffered by step parity; faces are symmetric between ranks, so a rank can
// only reach step t+2 after its neighbours finished reading step t.
// ---------------------------------------------------------------------------

__global__ void pack_faces_p2p(const ChunkDev* __restrict__ chunks,
                               const PackJob* __restrict__ jobs, double* const* __restrict__ peer_base,
                               int64_t half_elems, int32_t par, int32_t nz,
                               unsigned int* __restrict__ counter,
                               unsigned long long* const* __restrict__ peer_flags,
                               const int32_t* __restrict__ notify, int32_t n_notify,
                               int32_t my_rank, unsigned long long value) {
  const PackJob j = jobs[blockIdx.x];
  const ChunkDev& c = chunks[j.slot];
  const int f = blockIdx.y;
  const double* base = c.in + f * c.fstride;
  int64_t off = 0, es = 1;
  switch (j.side) {
    case kLeft: off = 0; es = c.pitch; break;
    case kRight: off = c.w - 1; es = c.pitch; break;
    case kTop: off = 0; es = 1; break;
    default: off = int64_t(c.h - 1) * c.pitch; es = 1; break;
  }
  double* out = peer_base[j.peer] + int64_t(par) * half_elems + j.rdst + int64_t(f) * nz * j.lenp;
  const int64_t n = int64_t(nz) * j.len;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t k = i / j.len, e = i - k * j.len;
    out[k * j.lenp + e] = base[off + k * c.kstride + e * es];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int total = gridDim.x * gridDim.y;
    if (atomicAdd(counter, 1u) == total - 1) {
      __threadfence_system();
      for (int i = 0; i < n_notify; ++i) st_release_sys(peer_flags[notify[i]] + my_rank, value);
      for (unsigned q = 0; q < gridDim.x; ++q)
        st_release_sys(peer_flags[jobs[q].peer] + jobs[q].rflag, value);
      *counter = 0u;  // next step's count (stream ordered)
    }
  }
}

// Chunk migration pulls: copy whole chunk arrays out of a peer GPU's slab (IPC
// mapping) over NVLink with SM loads, 16 bytes per thread per iteration.
struct CopyJob {
  const double* src;
  double* dst;
  int64_t n;  // doubles, even
};

__global__ void pull_chunks(const CopyJob* __restrict__ jobs) {
  const CopyJob j = jobs[blockIdx.y];
  const double2* __restrict__ s = reinterpret_cast<const double2*>(j.src);
  double2* __restrict__ d = reinterpret_cast<double2*>(j.dst);
  const int64_t n2 = j.n / 2;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2;
       i += int64_t(gridDim.x) * blockDim.x)
    d[i] = __ldcs(s + i);
}

// Diagnostic device timeline (OD_TIMELINE): one globaltimer stamp in stream order.
__global__ void stamp_time(unsigned long long* __restrict__ slot) { *slot = globaltimer_ns(); }
__global__ void fill_u32(unsigned* __restrict__ p, int n, unsigned v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}
__global__ void copy_u64(unsigned long long* __restrict__ dst,
                         const unsigned long long* __restrict__ src) { *dst = *src; }

__global__ void wait_halo(const unsigned long long* __restrict__ flags,
                          const int32_t* __restrict__ senders, int32_t n,
                          unsigned long long value, unsigned long long timeout_ns) {
  if (threadIdx.x == 0) wait_stamps(flags, senders, n, value, timeout_ns);
}

// ---------------------------------------------------------------------------
// Initial state: U[f][k][y][x] = H(seed, ((f*nz+k)*ny+gy)*nx+gx), A uses f = F.
// Padding columns are zeroed.
// ---------------------------------------------------------------------------
__global__ void init_chunk(double* __restrict__ u, double* __restrict__ a, int32_t w, int32_t h,
                           int32_t pitch, int32_t x0, int32_t y0, int32_t nx, int32_t ny,
                           int32_t nz, int32_t F, uint64_t seed) {
  const int64_t plane = int64_t(h) * pitch;
  const int64_t total = plane * nz * (F + 1);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t fk = i / plane;
    const int64_t r = i - fk * plane;
    const int yy = int(r / pitch), xx = int(r - int64_t(yy) * pitch);
    double v = 0.0;
    if (xx < w) {
      const uint64_t idx =
          ((uint64_t(fk) * uint64_t(ny) + uint64_t(y0 + yy)) * uint64_t(nx)) + uint64_t(x0 + xx);
      v = unit_hash(seed, idx);
    }
    if (fk < int64_t(F) * nz)
      u[i] = v;
    else
      a[i - int64_t(F) * nz * plane] = v;
  }
}

}  // namespace odb
