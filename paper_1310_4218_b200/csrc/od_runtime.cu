// B200 runtime of the over-decomposed column-update path: one instance per
// rank (= per GPU).  Replaces the modelled execution of the reference's
// Engine (engine.hpp:135-272) with real device work:
//
//   Engine::Engine      -> decomposition, block mapping, load field, chunk
//                          allocation, seeded initial state on the device
//   Engine::step_time   -> pack + NCCL halo exchange (cross-rank faces only),
//                          one batched Jacobi and one batched physics launch
//                          over the chunk table (Async), or per-chunk launches
//                          bracketed by cudaEvents / in-kernel per-chunk timers
//                          (Sync)
//   Engine::run_epoch   -> the same epoch policy on measured loads, then the
//                          migrate call moves chunk buffers between GPUs
//
// Neighbouring chunks on the same GPU read each other's boundary cells
// directly through per-face descriptors, so there is no halo copy at all
// inside a GPU; only faces that border another rank are packed and exchanged.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <tuple>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/overdeck_b200.h"
#include "od_capi_util.hpp"
#include "od_kernels.cuh"
#include "od_model.hpp"
#include "od_nccl.hpp"

namespace odb {

#define OD_CU(expr)                                                                      \
  do {                                                                                   \
    cudaError_t e__ = (expr);                                                            \
    if (e__ != cudaSuccess)                                                              \
      throw RuntimeFault(std::string("CUDA error ") + cudaGetErrorString(e__) + " in " + \
                         #expr);                                                         \
  } while (0)

#define OD_NC(expr)                                                                      \
  do {                                                                                   \
    ncclResult_t r__ = (expr);                                                           \
    if (r__ != ncclSuccess)                                                              \
      throw RuntimeFault(std::string("NCCL error ") + odb::nccl().GetErrorString(r__) + " in " + \
                         #expr);                                                         \
  } while (0)

static bool trace_on() {
  static const bool on = std::getenv("OD_TRACE") != nullptr;
  return on;
}
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

constexpr int kTX = 32, kTY = 8, kPrefetch = 4, kFusedPrefetch = 6;
constexpr int kGridMinBlocks = 4;  // column_step_grid CTAs per SM (<= 128 registers)
constexpr int kWsMinBlocks = 3;    // column_step_ws CTAs per SM

// Fused-tile width for a chunk of w x h columns: the shape (tw x 256/tw, two
// columns per thread, four row warps) that leaves the fewest idle lanes in the
// warps that hold any cell of the chunk; ties go to the wider tile.  64-wide
// chunks keep 64 x 4 tiles, cfg3's 32-wide chunks get 32 x 8, cfg1's 16 x 16,
// cfg2's 8 x 8 chunks one fully used warp of an 8 x 32 tile.
static int32_t tile_width(int32_t w, int32_t h) {
  int32_t best = 64;
  int64_t best_idle = -1;
  for (int32_t tw = 64; tw >= 8; tw >>= 1) {
    const int32_t th = 256 / tw, rpw = 64 / tw;  // rows per CTA, rows per warp
    const int64_t tiles_x = (w + tw - 1) / tw;
    const int64_t full_y = h / th, rem = h % th;
    const int64_t warps_y = full_y * kRowWarps + (rem + rpw - 1) / rpw;
    const int64_t idle = tiles_x * warps_y * 64 - int64_t(w) * h;
    if (best_idle < 0 || idle < best_idle) {
      best_idle = idle;
      best = tw;
    }
  }
  return best;
}

static int opposite(int d) { return d ^ 1; }

struct ChunkMem {
  int32_t vp = -1;
  Sub sub;
  int32_t pitch = 0;
  size_t bytes = 0;
  double* base = nullptr;
  double* u[2] = {nullptr, nullptr};
  double* a = nullptr;
  int64_t kstride() const { return int64_t(sub.h()) * pitch; }
};

struct StepRec {
  int32_t mode = kAsync;
  int32_t epoch_step = 0;          // the caller's label (reference semantics: any value)
  int32_t pos = 0;                 // position in the window: indexes the per-step device slots
  int64_t gstep = 0;               // global step index (st_.steps at launch)
  int ev_begin = -1, ev_end = -1;
  double host_launch_s = 0;
  int ns_row = -1;                  // TIMER: row of the per-chunk ns counters
  int chunk_ev0 = -1;               // EVENTS: first event of the per-chunk pairs
  int kev0 = -1, kev1 = -1;         // TIMER: events around the step's compute kernels
  bool ovl = false;                 // overlapped launch: wall from device stamps
  bool ovl_chained = false;         // ... and the previous step was overlapped too
  std::vector<int32_t> slot_vps;    // resident vps at launch time (slot order)
};

class Runtime {
 public:
  Runtime(const od_config& cfg, int rank, int world, int device, const uint8_t* nccl_id);
  ~Runtime();

  int32_t K() const { return int32_t(subs_.size()); }
  int32_t P() const { return cfg_.nodes * cfg_.procs_per_node; }
  const std::vector<int32_t>& mapping() const { return map_; }
  const std::vector<Sub>& subs() const { return subs_; }
  const Field2D& field() const { return field_; }
  std::vector<int32_t> classify() const;

  void step_api(int32_t mode, int32_t epoch_step, double* wall, od_sample* samples);
  void run_epoch(int32_t e, od_epoch_record* rec);
  void advance(int32_t n, int32_t* epochs_done);
  void advance_host(int32_t n, const double* host_c, int32_t n_fields, double* host_loads);
  void migrate(const std::vector<MoveRec>& plan);
  bool read_chunk(int32_t vp, double* u, double* a);
  void stats(od_rt_stats* s);
  void set_profiling(bool on) { profiling_ = on; }
  const std::vector<od_epoch_summary>& history() const { return history_; }
  void step_walls(int64_t first, int32_t n, double* out) const;
  void sync() { OD_CU(cudaStreamSynchronize(s0_)); }

 private:
  // processors (the reference's nodes x procs_per_node) are dealt to the GPUs
  // (ranks) in contiguous blocks; world == nodes gives node = GPU
  int rank_of_proc(int32_t p) const { return int(int64_t(p) * world_ / P()); }
  int rank_of_vp(int32_t v) const { return rank_of_proc(map_[v]); }
  int32_t nbr(int32_t v, int d) const;
  void set_shift(int32_t rows);
  void advance_advection(int32_t epoch, int32_t step);
  ChunkMem alloc_chunk(int32_t vp);
  void release_chunk(ChunkMem& m);
  void rebuild_tables();
  FaceDev edge_of(const ChunkMem& s, int side, int par) const;
  int new_event();
  void begin_window(bool allow_overlap = true);
  void launch_step(int32_t mode, int32_t epoch_step, bool host_io,
                   const double* host_field = nullptr, int staged_slot = -1);
  // waits for the window, gathers per-step walls and the K x S sample matrix
  void collect(std::vector<double>& walls, std::vector<double>& samples);
  struct EpochOut {
    std::vector<double> walls, loads, totals;
    std::vector<int32_t> map_before, classes;
    std::vector<MoveRec> plan;
    int32_t strategy = -1;
    double mig_s = 0, imb_before = 1, imb_after = 1;
  };
  void finish_epoch(int32_t e, int32_t steps, EpochOut& out);
  void require_no_open_window(const char* who) const;

  od_config cfg_;
  int rank_, world_, device_;
  std::vector<Sub> subs_;
  std::vector<int32_t> map_;
  Field2D base_, field_;
  int32_t shift_ = 0;
  int32_t global_step_ = 0, balance_calls_ = 0;
  int32_t parity_ = 0;
  // advance() state
  int32_t cur_epoch_ = 1, cur_step_ = 0;

  cudaStream_t s0_ = nullptr;
  unsigned int* d_counter_ = nullptr;
  ncclComm_t comm_ = nullptr;
  double* d_cbase_ = nullptr;   // base load field (device copy)
  // host_io path: the shifted field staged from pinned host memory every step
  // (double-buffered so the host fills one while the other is in flight) and
  // each step's per-chunk shares read back into a pinned row of h_loads_
  double* d_cstage_[2] = {nullptr, nullptr};
  double* h_cstage_[2] = {nullptr, nullptr};
  cudaEvent_t cstage_ev_[2] = {nullptr, nullptr};
  int cstage_cur_ = 0;
  unsigned long long* h_loads_ = nullptr;  // pinned [rows][2 * K]
  size_t h_loads_rows_ = 0;
  unsigned long long* h_loads_dst_ = nullptr;  // row for the step being launched
  // overlapped host-facing steps: per epoch step a mapped pinned field buffer
  // the step kernel reads straight over the host link, and mapped result rows
  std::vector<double*> h_ring_, d_ring_;
  unsigned long long* d_loads_map_ = nullptr;  // device view of h_loads_ (mapped)
  unsigned long long* d_loads_dst_ = nullptr;
  std::vector<ChunkMem> chunks_;  // indexed by vp; base == nullptr if not local
  std::multimap<size_t, double*> pool_;  // individually allocated (fallback) buffers
  double* slab_ = nullptr;                // preallocated chunk slots
  size_t slot_bytes_ = 0;
  std::vector<double*> free_slots_;
  size_t slab_slots_ = 0;
  void init_slab();
  std::vector<int32_t> resident_;  // slot -> vp
  std::vector<int32_t> tile_begin_, tile_count_;
  int32_t ntiles_ = 0;
  // fused-kernel tiles (tw x th, shape per chunk width: tile_shape), grouped by
  // chunk, and a heaviest-first copy for the batched launch
  std::vector<TileDev> tiles4_;          // grouped by chunk
  std::vector<int32_t> tile4_begin_, tile4_count_;
  TileDev* d_tiles4_ = nullptr;          // grouped (per-chunk launches)
  TileDev* d_tiles4s_[2] = {nullptr, nullptr};  // sorted, double buffered
  TileDev* h_tiles4s_[2] = {nullptr, nullptr};  // pinned staging
  cudaEvent_t tiles4s_ev_[2] = {nullptr, nullptr};
  size_t tiles4_cap_ = 0;
  int tiles4s_cur_ = 0;
  bool order_dirty_ = true;
  // A tile order refreshed inside an overlapped chain of step kernels (the
  // load field moves every step while a hotspot advects) is handed to the step
  // kernel in mapped pinned memory, one buffer per window position, so no copy
  // operation breaks the programmatic-dependent-launch chain; the next window
  // uploads the latest one to the device list.
  std::vector<TileDev*> h_oring_, d_oring_;
  size_t oring_cap_ = 0;
  int oring_pending_ = -1;             // window position of the live mapped order
  const TileDev* cur_tiles_ = nullptr;  // the list the step kernel reads
  int wave_grid_ = 0;  // tiles one launch keeps resident (SMs x CTAs per SM): column_step_grid
  int wave_ws_ = 0;    // the same for column_step_ws
  // equal-work tiles are dealt round-robin over the chunks in bands of band_
  // consecutive tiles of a chunk: y-neighbours start ~one CTA retirement apart,
  // so the halo rows they share are read within microseconds and hit L2.
  // cfg4 at N=1 (profiles/r2_tile_band_sweep.json): DRAM traffic per step
  // 68.3 GB (band 1) -> 62.6 (2) -> 59.7 (4) -> 59.0 GB (16) against 54.8 GB
  // algorithmic, step time unchanged (FP64-bound); the per-chunk load spread
  // among identical chunks grows 0.6 -> 1.0 -> 1.6 -> 12 % (CV): band 4.
  // OD_TILE_BAND overrides (diagnostic)
  int band_ = 4;
  int sms_ = 1;
  int pack_ctas_ = 0;  // CTAs of the step kernel that pack P2P halos (0: separate kernel)
  void refresh_tile_order(int mapped_pos = -1);
  // mode 5: the warp-specialised tile when a GPU holds less than one wave of
  // tiles (latency-bound), the interleaved tile otherwise; mode 7 always WS
  // mode 5 (default) and 7: the warp-specialised tile at every size (faster than
  // the interleaved one from 256 to 4096 tiles per GPU, profiles/r2_ws_threshold.json)
  bool use_ws() const {
    return cfg_.overlap == 7 || cfg_.overlap == 5;
  }
  int32_t last_kernel_ = 0;  // OD_KERNEL_* of the last step kernel launched
  // cross-step overlap of the mode-5 step kernels (PDL + per-tile stamps;
  // OD_OVERLAP=0 disables): tile -> same-GPU tiles whose cells it reads (itself first),
  // pack job -> tiles holding its face cells; per-tile completed-step stamps
  bool overlap_ = false;
  std::vector<int32_t> deps_;  // [off (n+1) | idx | joff (nj+1) | jidx]
  int32_t* d_deps_ = nullptr;
  size_t d_deps_cap_ = 0;
  int32_t dep_idx_at_ = 0, dep_joff_at_ = 0, dep_jidx_at_ = 0;
  unsigned* d_done_ = nullptr;
  size_t d_done_cap_ = 0;
  unsigned long long* d_stepend_ = nullptr;  // [window steps + 1]: start, end of each step
  unsigned* d_pcnt_ = nullptr;                // [window steps][2] fused-pack counters
  unsigned* d_jcnt_ = nullptr;                // [window steps][4 K] per-strip field counts
  unsigned* d_jcnt1_ = nullptr;               // [4 K] the same for a step outside a window
  int64_t* d_mig_off_ = nullptr;              // migration: [world + 1][K] slab offsets
  CopyJob* d_mig_jobs_ = nullptr;             // migration: pull jobs (at most 2 K)
  int32_t* d_mig_one_ = nullptr;              // migration: ordering all-reduce word
  int32_t win_cap_ = 0;
  bool win_overlap_ = false;  // this window's steps ran overlapped
  void build_step_deps();
  // host caches keyed on the load-field generation (set_shift bumps it)
  uint64_t field_gen_ = 0;
  std::vector<std::vector<double>> tile_work_;  // per vp, per tile of the chunk
  std::vector<uint64_t> tile_work_gen_;
  mutable std::vector<int32_t> classes_;
  mutable uint64_t classes_gen_ = ~0ull;
  ChunkDev* d_chunks_[2] = {nullptr, nullptr};
  // TMA tensor maps of the full tiles' planes, per parity and slot: [main box,
  // own row, top-face row source, bottom-face row source].  Opt-in: OD_TMA=1
  // stages 64-wide full tiles through TMA, OD_TMA=2 every width.  Default off:
  // at cfg4 the TMA-staged kernel reads 10 % more DRAM (L2 hit rate 12.5 % vs
  // 43 %, independent of the L2 promotion) and takes 3.8 % more cycles than the
  // cp.async ring; at free clocks it runs at higher SM clocks for the same step
  // time (profiles/r2_tma_vs_cpasync.json).  OD_TMA_L2: promotion experiment.
  bool tma_on_ = false;
  int tma_min_width_ = 64;
  PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_ = nullptr;
  CUtensorMap* d_tmaps_ = nullptr;
  size_t d_tmaps_cap_ = 0;
  void build_tensor_maps(std::vector<ChunkDev>& tab, int par, const std::vector<int32_t>& slot_of);
  size_t d_chunks_cap_[2] = {0, 0};
  TileDev* d_tiles_ = nullptr;
  size_t d_tiles_cap_ = 0;
  // exchange
  std::vector<PackJob> jobs_;
  PackJob* d_jobs_ = nullptr;
  size_t d_jobs_cap_ = 0;
  std::vector<int64_t> send_off_, send_cnt_, recv_off_, recv_cnt_;  // per peer, elements
  double* d_send_ = nullptr;
  double* d_recv_ = nullptr;
  // NVLink peer-memory halo exchange (CUDA IPC), default for world > 1
  bool p2p_ = false;
  int64_t recv_half_ = 0;  // elements per parity half of d_recv_ (p2p)
  // [world] step published by each sender, then [4 K] per receiving chunk face
  unsigned long long* d_flags_ = nullptr;
  std::vector<double*> peer_recv_;
  std::vector<double*> peer_slab_;  // every rank's chunk slab (IPC), for migration pulls
  bool peer_slabs_ok_ = false;
  // column_step_ws: spread grids of at most one tile per SM (see launch_step)
  static constexpr size_t kWsSpreadSmem = 150 * 1024;
  bool ws_spread_ = true;
  std::vector<unsigned long long*> peer_flags_;
  double** d_peer_base_ = nullptr;
  unsigned long long** d_peer_flags_ = nullptr;
  unsigned int* d_pack_counter_ = nullptr;
  int32_t* d_notify_ = nullptr;   // ranks this rank sends to
  int32_t* d_senders_ = nullptr;  // ranks that send to this rank
  int32_t n_notify_ = 0, n_senders_ = 0;
  void alloc_comm_buffers();
  void setup_p2p();
  size_t send_cap_ = 0, recv_cap_ = 0;
  std::vector<std::array<int64_t, 4>> recv_face_off_;  // per slot
  // measurement
  std::vector<cudaEvent_t> events_;
  int ev_used_ = 0;
  std::vector<StepRec> window_;
  unsigned long long* d_ns_ = nullptr;  // [rows][cap_slots]
  int ns_rows_ = 0, ns_cols_ = 0, ns_used_ = 0;
  unsigned long long* d_trips_ = nullptr;
  double* d_gather_ = nullptr;
  size_t gather_cap_ = 0;
  // diagnostic device timeline (env OD_TIMELINE=<path prefix>): per step,
  // globaltimer stamps at step begin, after the halo pack, before and after
  // the step kernel; written to <prefix>.rank<r>.txt at destruction
  unsigned long long* d_tl_ = nullptr;
  int tl_cap_ = 0, tl_n_ = 0;
  void tl_mark(int k) {
    if (d_tl_ && tl_n_ < tl_cap_) stamp_time<<<1, 1, 0, s0_>>>(d_tl_ + size_t(tl_n_) * 5 + k);
  }
  void tl_dump();
  double tr_drained_ = 0;  // OD_TRACE: host time the stream last drained
  // diagnostic share-clock event log of one step (env OD_TILELOG=<path>, OD_TILELOG_STEP=<n>)
  ShareEvent* d_slog_ = nullptr;
  unsigned slog_cap_ = 0;
  long slog_step_ = -1;
  void slog_arm(bool on);
  void slog_dump();
  unsigned long long* tl_wait() {
    return d_tl_ && tl_n_ < tl_cap_ ? d_tl_ + size_t(tl_n_) * 5 + 4 : nullptr;
  }
  // stats
  bool profiling_ = false;
  std::vector<std::pair<int, int>> prof_j_, prof_p_, prof_pack_, prof_x_, prof_f_;
  od_rt_stats st_{};
  std::vector<double> step_wall_;  // by global step index (NaN until collected)
  Capacity capacity_;  // per-GPU chunk-data bins (cfg.capacity_mib > 0)
  std::vector<od_epoch_summary> history_;
};

// --------------------------------------------------------------- lifecycle --

Runtime::Runtime(const od_config& cfg, int rank, int world, int device, const uint8_t* nccl_id)
    : cfg_(cfg), rank_(rank), world_(world), device_(device) {
  // ExperimentConfig::validate (engine.hpp:62-83) + B200 constraints
  if (cfg.nodes < 1) throw ValidationError("cluster.nodes must be >= 1");
  if (cfg.procs_per_node < 1) throw ValidationError("cluster.procs_per_node must be >= 1");
  check_domain(cfg.nx, cfg.ny, cfg.nz, cfg.fields);
  if (cfg.fields < 1) throw ValidationError("the B200 path needs fields >= 1 (physics reads field 0)");
  if (cfg.async_steps < 0) throw ValidationError("window.async_steps must be >= 0");
  if (cfg.sync_steps < 1) throw ValidationError("window.sync_steps must be >= 1");
  if (cfg.adv_total_shift_rows < 0) throw ValidationError("advection.total_shift_rows must be >= 0");
  if (cfg.adv_epoch < 0) throw ValidationError("advection.epoch must be >= 0");
  if (cfg.adv_duration_steps < 1) throw ValidationError("advection.duration_steps must be >= 1");
  if (cfg.trigger_threshold < 1.0) throw ValidationError("policy.trigger_threshold must be >= 1");
  if (cfg.refine_tolerance < 0.0) throw ValidationError("policy.refine_tolerance must be >= 0");
  if (cfg.epochs < 1) throw ValidationError("epochs must be >= 1");
  if (cfg.kx < 1 || cfg.ky < 1) throw ValidationError("decomposition counts must be >= 1");
  if (cfg.decomposition_kind == OD_ONE_D && cfg.kx != 1)
    throw ValidationError("1d decomposition requires kx = 1");
  if (cfg.decomposition_kind != OD_ONE_D && cfg.decomposition_kind != OD_TWO_D)
    throw ValidationError("unknown decomposition kind");
  if (cfg.kx * cfg.ky < cfg.nodes * cfg.procs_per_node)
    throw ValidationError("vp count must be >= processor count");
  if (cfg.heavy_value < cfg.light_value || cfg.light_value < 1)
    throw ValidationError("load values require heavy >= light >= 1");
  if (cfg.first_call_strategy < 0 || cfg.first_call_strategy > 2 ||
      cfg.later_call_strategy < 0 || cfg.later_call_strategy > 2)
    throw ValidationError("unknown strategy");
  if (cfg.n_inner < 0) throw ValidationError("n_inner must be >= 0");
  if (cfg.overlap != 0 && cfg.overlap != 4 && cfg.overlap != 5 && cfg.overlap != 7)
    throw ValidationError("unknown kernel mode (overlap): 0 separate, 4 interleaved tiles, "
                          "5 automatic, 7 warp-specialised tiles");
  if (cfg.measure != OD_MEASURE_EVENTS && cfg.measure != OD_MEASURE_TIMER &&
      cfg.measure != OD_MEASURE_TIMER_RAW && cfg.measure != OD_MEASURE_OPS)
    throw ValidationError("unknown measurement mode");
  if (world < 1 || world > cfg.nodes * cfg.procs_per_node)
    throw ValidationError("world size must be between 1 and the processor count "
                          "(cluster.nodes x cluster.procs_per_node)");
  if (rank < 0 || rank >= world) throw ValidationError("rank out of range");
  if (world > 1 && !nccl_id) throw ValidationError("multi-rank runtime needs an NCCL id");

  subs_ = cfg.decomposition_kind == OD_ONE_D ? strips_1d(cfg.nx, cfg.ny, cfg.ky)
                                             : tiles_2d(cfg.nx, cfg.ny, cfg.kx, cfg.ky);
  map_ = block_mapping(K(), P());
  // static_node0 heats the VPs initially homed on the reference's node 0
  // (workload.hpp:160-181 via engine.hpp:141-148), whatever GPU holds them
  std::vector<Sub> node0;
  for (int32_t v = 0; v < K(); ++v)
    if (map_[v] / cfg.procs_per_node == 0) node0.push_back(subs_[v]);
  base_ = make_load_field(cfg.nx, cfg.ny, Pattern(cfg.pattern), cfg.heavy_value,
                          cfg.light_value, node0);
  if (cfg.capacity_mib < 0) throw ValidationError("capacity_mib must be >= 0");
  if (cfg.capacity_mib > 0) {
    // one bin per GPU; a chunk's footprint is its device allocation (U^t,
    // U^{t+1}, A with the pitch padding)
    capacity_.bin_cap.assign(world_, int64_t(cfg.capacity_mib) << 20);
    capacity_.bin_of_proc.resize(P());
    for (int32_t p = 0; p < P(); ++p) capacity_.bin_of_proc[p] = rank_of_proc(p);
    capacity_.vp_bytes.resize(K());
    std::vector<int64_t> used(world_, 0);
    for (int32_t v = 0; v < K(); ++v) {
      const int64_t plane = int64_t(subs_[v].h()) * ((subs_[v].w() + 15) / 16 * 16);
      capacity_.vp_bytes[v] = (2 * plane * cfg.nz * cfg.fields + plane * cfg.nz) * 8;
      used[rank_of_vp(v)] += capacity_.vp_bytes[v];
    }
    for (int q = 0; q < world_; ++q)
      if (used[q] > capacity_.bin_cap[q])
        throw ValidationError("capacity_mib is below the initial chunk data of GPU " +
                              std::to_string(q) + " (" + std::to_string(used[q] >> 20) + " MiB)");
  }

  OD_CU(cudaSetDevice(device_));
  OD_CU(cudaStreamCreateWithFlags(&s0_, cudaStreamNonBlocking));
  if (std::getenv("OD_TILELOG")) {
    slog_cap_ = 1u << 20;
    slog_step_ = std::getenv("OD_TILELOG_STEP") ? std::atol(std::getenv("OD_TILELOG_STEP")) : 19;
    OD_CU(cudaMalloc(&d_slog_, size_t(slog_cap_) * sizeof(ShareEvent)));
  }
  if (std::getenv("OD_TIMELINE")) {
    tl_cap_ = 8192;
    OD_CU(cudaMalloc(&d_tl_, size_t(tl_cap_) * 5 * sizeof(unsigned long long)));
    OD_CU(cudaMemset(d_tl_, 0, size_t(tl_cap_) * 5 * sizeof(unsigned long long)));
  }
  {
    int sms = 0;
    OD_CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    sms_ = sms;
    // cross-step overlap of the step kernels unless OD_OVERLAP=0 (diagnostic)
    overlap_ = !(std::getenv("OD_OVERLAP") && std::string(std::getenv("OD_OVERLAP")) == "0");
    // P2P halos: the step kernel's first CTAs pack the strips (OD_PACK_CTAS=0:
    // a separate pack kernel ahead of the step kernel)
    pack_ctas_ = std::getenv("OD_PACK_CTAS") ? std::atoi(std::getenv("OD_PACK_CTAS")) : sms;
    if (const char* b = std::getenv("OD_TILE_BAND")) band_ = std::max(1, std::atoi(b));
    if (const char* t = std::getenv("OD_TMA")) {
      tma_on_ = std::atoi(t) > 0;
      if (std::atoi(t) == 2) tma_min_width_ = 8;
    }
    if (tma_on_) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
              cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
        throw RuntimeFault("cuTensorMapEncodeTiled unavailable (unset OD_TMA to stage with cp.async)");
      encode_tiled_ = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    OD_CU(cudaMalloc(&d_counter_, 4 * sizeof(unsigned int)));  // [tiles, pack next, pack done]
    int per_sm = 0;
    OD_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, column_step_grid<kFusedPrefetch, false, kGridMinBlocks>, 32 * kRowWarps, 0));
    wave_grid_ = sms * std::max(per_sm, 1);
    OD_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, column_step_ws<kFusedPrefetch, false, kWsMinBlocks>, 64 * kRowWarps, 0));
    wave_ws_ = sms * std::max(per_sm, 1);
  }
  if (world_ > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    OD_NC(odb::nccl().CommInitRank(&comm_, world_, id, rank_));
    // NCCL connects peers lazily on first use; pay that here, not inside the
    // first exchange/migration/gather of the run: one all-gather and one
    // send/recv with every peer
    double* tmp = nullptr;
    OD_CU(cudaMalloc(&tmp, sizeof(double) * 2 * (world_ + 1)));
    OD_CU(cudaMemset(tmp, 0, sizeof(double) * 2 * (world_ + 1)));
    OD_NC(odb::nccl().AllGather(tmp, tmp + 1, 1, ncclFloat64, comm_, s0_));
    OD_NC(odb::nccl().GroupStart());
    for (int q = 0; q < world_; ++q) {
      if (q == rank_) continue;
      OD_NC(odb::nccl().Send(tmp, 1, ncclFloat64, q, comm_, s0_));
      OD_NC(odb::nccl().Recv(tmp + world_ + 1 + q, 1, ncclFloat64, q, comm_, s0_));
    }
    OD_NC(odb::nccl().GroupEnd());
    OD_CU(cudaStreamSynchronize(s0_));
    cudaFree(tmp);
  }
  const size_t cbytes = base_.c.size() * sizeof(double);
  OD_CU(cudaMalloc(&d_cbase_, cbytes));
  OD_CU(cudaMemcpy(d_cbase_, base_.c.data(), cbytes, cudaMemcpyHostToDevice));
  set_shift(0);

  init_slab();
  if (world_ > 1) {
    const char* hm = std::getenv("OD_HALO");
    p2p_ = !(hm && std::string(hm) == "nccl");
    alloc_comm_buffers();
    if (p2p_) setup_p2p();
  }
  chunks_.resize(K());
  for (int32_t v = 0; v < K(); ++v) {
    if (rank_of_vp(v) != rank_) continue;
    chunks_[v] = alloc_chunk(v);
    const ChunkMem& m = chunks_[v];
    init_chunk<<<296, 256, 0, s0_>>>(m.u[0], m.a, m.sub.w(), m.sub.h(), m.pitch, m.sub.x0,
                                     m.sub.y0, cfg.nx, cfg.ny, cfg.nz, cfg.fields, cfg.seed);
    OD_CU(cudaGetLastError());
    ++st_.kernel_launches;
  }
  rebuild_tables();
  OD_CU(cudaStreamSynchronize(s0_));
}

void Runtime::slog_arm(bool on) {
  ShareEvent* p = on ? d_slog_ : nullptr;
  unsigned zero = 0;
  OD_CU(cudaMemcpyToSymbolAsync(g_share_log, &p, sizeof(p), 0, cudaMemcpyHostToDevice, s0_));
  if (on) {
    OD_CU(cudaMemcpyToSymbolAsync(g_share_log_n, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s0_));
    OD_CU(cudaMemcpyToSymbolAsync(g_share_log_cap, &slog_cap_, sizeof(slog_cap_), 0,
                                  cudaMemcpyHostToDevice, s0_));
  }
}

void Runtime::slog_dump() {
  const char* path = std::getenv("OD_TILELOG");
  if (!d_slog_ || !path) return;
  unsigned n = 0;
  if (cudaMemcpyFromSymbol(&n, g_share_log_n, sizeof(n)) != cudaSuccess) return;
  n = std::min(n, slog_cap_);
  std::vector<ShareEvent> h(n);
  if (n && cudaMemcpy(h.data(), d_slog_, n * sizeof(ShareEvent), cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  const std::string p = std::string(path) + ".rank" + std::to_string(rank_) + ".txt";
  if (FILE* f = std::fopen(p.c_str(), "w")) {
    for (const auto& e : h)
      std::fprintf(f, "%llu %.3f %d %d %d %d\n", e.t, e.v, e.n, e.tag, e.sm, e.delta);
    std::fclose(f);
  }
}

void Runtime::tl_dump() {
  const char* pre = std::getenv("OD_TIMELINE");
  if (!d_tl_ || !pre || tl_n_ == 0) return;
  std::vector<unsigned long long> h(size_t(tl_n_) * 5);
  if (cudaMemcpy(h.data(), d_tl_, h.size() * sizeof(unsigned long long),
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  const std::string path = std::string(pre) + ".rank" + std::to_string(rank_) + ".txt";
  if (FILE* f = std::fopen(path.c_str(), "w")) {
    for (int i = 0; i < tl_n_; ++i)
      std::fprintf(f, "%d %llu %llu %llu %llu %llu\n", i, h[5 * i], h[5 * i + 1], h[5 * i + 2],
                   h[5 * i + 3], h[5 * i + 4]);
    std::fclose(f);
  }
}

Runtime::~Runtime() {
  cudaSetDevice(device_);
  if (s0_) cudaStreamSynchronize(s0_);
  tl_dump();
  cudaFree(d_tl_);
  cudaFree(d_deps_);
  cudaFree(d_done_);
  cudaFree(d_stepend_);
  cudaFree(d_pcnt_);
  cudaFree(d_jcnt_);
  cudaFree(d_jcnt1_);
  cudaFree(d_mig_off_);
  cudaFree(d_mig_jobs_);
  cudaFree(d_mig_one_);
  slog_dump();
  cudaFree(d_slog_);
  for (auto& m : chunks_)
    if (m.base && !(slab_ && m.base >= slab_ &&
                    m.base < slab_ + slab_slots_ * (slot_bytes_ / sizeof(double))))
      cudaFree(m.base);
  cudaFree(slab_);
  for (auto& kv : pool_) cudaFree(kv.second);
  for (auto e : events_) cudaEventDestroy(e);
  cudaFree(d_cbase_);
  for (int b = 0; b < 2; ++b) {
    cudaFree(d_cstage_[b]);
    if (h_cstage_[b]) cudaFreeHost(h_cstage_[b]);
    if (cstage_ev_[b]) cudaEventDestroy(cstage_ev_[b]);
  }
  if (h_loads_) cudaFreeHost(h_loads_);
  for (double* p : h_ring_) cudaFreeHost(p);
  for (TileDev* p : h_oring_) cudaFreeHost(p);
  cudaFree(d_chunks_[0]);
  cudaFree(d_chunks_[1]);
  cudaFree(d_tmaps_);
  cudaFree(d_tiles_);
  cudaFree(d_tiles4_);
  for (int b = 0; b < 2; ++b) {
    cudaFree(d_tiles4s_[b]);
    if (h_tiles4s_[b]) cudaFreeHost(h_tiles4s_[b]);
    if (tiles4s_ev_[b]) cudaEventDestroy(tiles4s_ev_[b]);
  }
  cudaFree(d_jobs_);
  cudaFree(d_send_);
  cudaFree(d_recv_);
  cudaFree(d_ns_);
  cudaFree(d_trips_);
  cudaFree(d_gather_);
  for (int q = 0; q < int(peer_recv_.size()); ++q) {
    if (q == rank_) continue;
    if (peer_recv_[q]) cudaIpcCloseMemHandle(peer_recv_[q]);
    if (q < int(peer_slab_.size()) && peer_slab_[q]) cudaIpcCloseMemHandle(peer_slab_[q]);
    if (peer_flags_[q]) cudaIpcCloseMemHandle(peer_flags_[q]);
  }
  cudaFree(d_flags_);
  cudaFree(d_peer_base_);
  cudaFree(d_peer_flags_);
  cudaFree(d_pack_counter_);
  cudaFree(d_notify_);
  cudaFree(d_senders_);
  if (comm_) odb::nccl().CommDestroy(comm_);
  cudaFree(d_counter_);
  if (s0_) cudaStreamDestroy(s0_);
}

// ------------------------------------------------------------------ model --

int32_t Runtime::nbr(int32_t v, int d) const {
  return chunk_neighbor(cfg_.decomposition_kind, cfg_.kx, cfg_.ky, v, d);
}

void Runtime::set_shift(int32_t rows) {
  shift_ = rows;
  field_ = shift_rows_down(base_, rows % cfg_.ny);
  ++field_gen_;
  order_dirty_ = true;
}

// Heaviest tiles first (longest-processing-time order) for the batched step
// kernel: estimated work = physics units + Jacobi cells, from the current field.
void Runtime::refresh_tile_order(int mapped_pos) {
  const size_t n = tiles4_.size();
  if (n == 0) return;
  // (group, -work, tile index within its chunk, tile): equal-work tiles are
  // dealt round-robin over the chunks, so each chunk's tiles meet every queue
  // position (and with it every issue priority on the SM: the warp scheduler
  // favours older CTAs) and the per-chunk measurements average over them
  std::vector<std::tuple<double, int32_t, int32_t>> key(n);
  const double jac = 2.0 * cfg_.nz * cfg_.fields;  // a Jacobi cell ~ 2 micro-steps
  if (tile_work_.size() != size_t(K())) {
    tile_work_.assign(K(), {});
    tile_work_gen_.assign(K(), ~0ull);
  }
  for (size_t t = 0; t < n; ++t) {
    const TileDev& td = tiles4_[t];
    const int32_t vp = resident_[td.slot];
    const size_t local = t - size_t(tile4_begin_[td.slot]);
    if (tile_work_gen_[vp] != field_gen_) {
      // the work of every tile of this chunk under the current load field
      tile_work_gen_[vp] = field_gen_;
      auto& tw = tile_work_[vp];
      tw.assign(size_t(tile4_count_[td.slot]), 0.0);
      const Sub& s = subs_[vp];
      for (int32_t j = 0; j < tile4_count_[td.slot]; ++j) {
        const TileDev& tj = tiles4_[tile4_begin_[td.slot] + j];
        const int32_t x0 = s.x0 + tj.tx0, x1 = std::min(s.x1, x0 + tj.tw);
        const int32_t y0 = s.y0 + tj.ty0, y1 = std::min(s.y1, y0 + tj.th);
        double w = 0;
        for (int32_t y = y0; y < y1; ++y)
          for (int32_t x = x0; x < x1; ++x) {
            const int32_t T = int32_t(std::floor(double(cfg_.nz) * field_.at(x, y))) - 1;
            w += double(T > 0 ? T : 0) * (cfg_.n_inner + 1) + jac;
          }
        tw[j] = w;
      }
    }
    const double w = tile_work_[vp][local];
    key[t] = {-w, (int32_t(t) - tile4_begin_[td.slot]) / band_, int32_t(t)};
  }
  std::sort(key.begin(), key.end());
  if (p2p_ && n_senders_ > 0) {
    // with peer-memory halos the neighbours' strips of this step land while the
    // kernel runs: the first wave (one tile per CTA) takes the heaviest tiles
    // that read no remote strip; everything after it stays in heaviest-first
    // order (deferring all boundary tiles to the end would put heavy migrated
    // chunks -- typically boundary after a rebalance -- into the tail).
    // Measured 5-7 % faster at 4 GPUs on cfg4 than plain heaviest-first.
    std::vector<std::tuple<double, int32_t, int32_t>> front, rest;
    front.reserve(n);
    rest.reserve(n);
    const size_t wave = size_t(use_ws() ? wave_ws_ : wave_grid_);
    for (const auto& k : key)
      (front.size() < wave && !(tiles4_[std::get<2>(k)].pad & 1) ? front : rest)
          .push_back(k);
    front.insert(front.end(), rest.begin(), rest.end());
    key.swap(front);
  }
  order_dirty_ = false;
  if (mapped_pos >= 0 && mapped_pos < int(h_oring_.size()) && n <= oring_cap_) {
    // inside an overlapped chain: the kernel reads this order from mapped memory
    for (size_t t = 0; t < n; ++t) h_oring_[mapped_pos][t] = tiles4_[std::get<2>(key[t])];
    cur_tiles_ = d_oring_[mapped_pos];
    oring_pending_ = mapped_pos;
    return;
  }
  const int b = tiles4s_cur_ ^ 1;
  OD_CU(cudaEventSynchronize(tiles4s_ev_[b]));  // previous upload from this buffer done
  for (size_t t = 0; t < n; ++t) h_tiles4s_[b][t] = tiles4_[std::get<2>(key[t])];
  OD_CU(cudaMemcpyAsync(d_tiles4s_[b], h_tiles4s_[b], n * sizeof(TileDev),
                        cudaMemcpyHostToDevice, s0_));
  OD_CU(cudaEventRecord(tiles4s_ev_[b], s0_));
  tiles4s_cur_ = b;
  cur_tiles_ = d_tiles4s_[b];
  oring_pending_ = -1;
}

// engine.hpp:323-336
void Runtime::advance_advection(int32_t epoch, int32_t step) {
  if (cfg_.adv_epoch == 0 || cfg_.adv_total_shift_rows == 0) return;
  int32_t target = shift_;
  if (epoch > cfg_.adv_epoch) {
    target = cfg_.adv_total_shift_rows;
  } else if (epoch == cfg_.adv_epoch) {
    const int32_t k = std::min(step + 1, cfg_.adv_duration_steps);
    target = int32_t(std::lround(double(cfg_.adv_total_shift_rows) * k / cfg_.adv_duration_steps));
  }
  if (target != shift_) set_shift(target);
}

// engine.hpp:281-287
std::vector<int32_t> Runtime::classify() const {
  if (classes_gen_ == field_gen_) return classes_;
  const double mid = 0.5 * (cfg_.heavy_value + cfg_.light_value);
  std::vector<int32_t> out(K());
  for (int32_t v = 0; v < K(); ++v) out[v] = field_.mean_over(subs_[v]) > mid ? kHeavy : kLight;
  classes_ = out;
  classes_gen_ = field_gen_;
  return out;
}

// ----------------------------------------------------------------- memory --

// One slab of equal chunk slots, sized at creation for the resident chunks plus
// migration headroom (bounded by free HBM), so migrations do not cudaMalloc.
void Runtime::init_slab() {
  if (const char* e = std::getenv("OD_WS_SPREAD")) ws_spread_ = std::atoi(e) != 0;
  if (ws_spread_) {
    OD_CU(cudaFuncSetAttribute(column_step_ws<kFusedPrefetch, true, kWsMinBlocks>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWsSpreadSmem)));
    OD_CU(cudaFuncSetAttribute(column_step_ws<kFusedPrefetch, false, kWsMinBlocks>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWsSpreadSmem)));
  }
  for (const Sub& sb : subs_) {
    const size_t plane = size_t(sb.h()) * ((sb.w() + 15) / 16 * 16);
    const size_t b = (2 * plane * cfg_.nz * cfg_.fields + plane * cfg_.nz) * sizeof(double);
    slot_bytes_ = std::max(slot_bytes_, (b + 4095) / 4096 * 4096);
  }
  size_t resident = 0;
  for (int32_t v = 0; v < K(); ++v) resident += rank_of_vp(v) == rank_;
  size_t want = world_ == 1 ? resident : std::min<size_t>(K(), 2 * resident + 4);
  size_t free_b = 0, total_b = 0;
  OD_CU(cudaMemGetInfo(&free_b, &total_b));
  const size_t margin = size_t(6) << 30;
  const size_t fit = free_b > margin ? (free_b - margin) / slot_bytes_ : 0;
  want = std::max(resident, std::min(want, fit));
  if (want == 0) return;
  OD_CU(cudaMalloc(&slab_, want * slot_bytes_));
  slab_slots_ = want;
  free_slots_.reserve(want);
  for (size_t i = want; i-- > 0;) free_slots_.push_back(slab_ + i * (slot_bytes_ / sizeof(double)));
}

ChunkMem Runtime::alloc_chunk(int32_t vp) {
  ChunkMem m;
  m.vp = vp;
  m.sub = subs_[vp];
  m.pitch = (m.sub.w() + 15) / 16 * 16;
  const size_t plane = size_t(m.sub.h()) * m.pitch;
  const size_t field_elems = plane * cfg_.nz * cfg_.fields;
  m.bytes = (2 * field_elems + plane * cfg_.nz) * sizeof(double);
  if (!free_slots_.empty() && m.bytes <= slot_bytes_) {
    m.base = free_slots_.back();
    free_slots_.pop_back();
  } else {
    auto it = pool_.find(m.bytes);
    if (it != pool_.end()) {
      m.base = it->second;
      pool_.erase(it);
    } else {
      OD_CU(cudaMalloc(&m.base, m.bytes));
    }
  }
  m.u[0] = m.base;
  m.u[1] = m.base + field_elems;
  m.a = m.base + 2 * field_elems;
  return m;
}

void Runtime::release_chunk(ChunkMem& m) {
  if (m.base) {
    const bool slab = slab_ && m.base >= slab_ &&
                      m.base < slab_ + slab_slots_ * (slot_bytes_ / sizeof(double));
    if (slab)
      free_slots_.push_back(m.base);
    else
      pool_.emplace(m.bytes, m.base);
  }
  m = ChunkMem();
}

FaceDev Runtime::edge_of(const ChunkMem& s, int side, int par) const {
  FaceDev f;
  const double* b = s.u[par];
  f.lo = b;
  f.hi = b + s.kstride() * cfg_.nz * cfg_.fields;
  f.fs = s.kstride() * cfg_.nz;
  f.ks = s.kstride();
  switch (side) {
    case kLeft: f.p = b; f.es = s.pitch; break;
    case kRight: f.p = b + (s.sub.w() - 1); f.es = s.pitch; break;
    case kTop: f.p = b; f.es = 1; break;
    default: f.p = b + int64_t(s.sub.h() - 1) * s.pitch; f.es = 1; break;
  }
  return f;
}

template <typename T>
static void upload(T*& dptr, size_t& cap, const std::vector<T>& h) {
  if (h.size() > cap) {
    cudaFree(dptr);
    dptr = nullptr;
    cap = std::max<size_t>(h.size() * 2, 16);
    OD_CU(cudaMalloc(&dptr, cap * sizeof(T)));
  }
  if (!h.empty()) OD_CU(cudaMemcpy(dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

void Runtime::build_step_deps() {
  const size_t n = tiles4_.size();
  std::vector<int32_t> slot_of(K(), -1);
  for (size_t i = 0; i < resident_.size(); ++i) slot_of[resident_[i]] = int32_t(i);
  struct Rect {
    int32_t x0, x1, y0, y1;
  };
  auto rect = [&](const TileDev& t) {
    const Sub& s = subs_[resident_[t.slot]];
    return Rect{s.x0 + t.tx0, std::min(s.x1, s.x0 + t.tx0 + t.tw), s.y0 + t.ty0,
                std::min(s.y1, s.y0 + t.ty0 + t.th)};
  };
  auto overlaps = [](const Rect& a, const Rect& b) {
    return a.x0 < b.x1 && b.x0 < a.x1 && a.y0 < b.y1 && b.y0 < a.y1;
  };
  std::vector<int32_t> off(n + 1, 0), idx;
  for (size_t t = 0; t < n; ++t) {
    const TileDev& td = tiles4_[t];
    off[t] = int32_t(idx.size());
    idx.push_back(int32_t(t));
    const Rect r = rect(td);
    // the four one-cell halo strips of the tile
    const Rect halo[4] = {{r.x0 - 1, r.x0, r.y0, r.y1}, {r.x1, r.x1 + 1, r.y0, r.y1},
                          {r.x0, r.x1, r.y0 - 1, r.y0}, {r.x0, r.x1, r.y1, r.y1 + 1}};
    const int32_t v = resident_[td.slot];
    // candidate chunks: the tile's own and its four neighbours on this GPU
    int32_t cand[5] = {td.slot, -1, -1, -1, -1};
    for (int d = 0; d < 4; ++d) {
      const int32_t nb = nbr(v, d);
      cand[d + 1] = nb >= 0 ? slot_of[nb] : -1;
    }
    for (int c = 0; c < 5; ++c) {
      if (cand[c] < 0) continue;
      const int32_t j0 = tile4_begin_[cand[c]], j1 = j0 + tile4_count_[cand[c]];
      for (int32_t j = j0; j < j1; ++j) {
        if (size_t(j) == t) continue;
        const Rect q = rect(tiles4_[j]);
        bool hit = false;
        for (int h = 0; h < 4 && !hit; ++h) hit = overlaps(halo[h], q);
        if (hit && std::find(idx.begin() + off[t], idx.end(), j) == idx.end()) idx.push_back(j);
      }
    }
  }
  off[n] = int32_t(idx.size());
  std::vector<int32_t> joff(jobs_.size() + 1, 0), jidx;
  for (size_t jb = 0; jb < jobs_.size(); ++jb) {
    joff[jb] = int32_t(jidx.size());
    const PackJob& pj = jobs_[jb];
    const Sub& s = subs_[resident_[pj.slot]];
    const int32_t j0 = tile4_begin_[pj.slot], j1 = j0 + tile4_count_[pj.slot];
    for (int32_t j = j0; j < j1; ++j) {
      const TileDev& tj = tiles4_[j];
      const bool edge = (pj.side == kLeft && tj.tx0 == 0) ||
                        (pj.side == kRight && tj.tx0 + tj.tw >= s.w()) ||
                        (pj.side == kTop && tj.ty0 == 0) ||
                        (pj.side == kBottom && tj.ty0 + tj.th >= s.h());
      if (edge) jidx.push_back(j);
    }
  }
  joff[jobs_.size()] = int32_t(jidx.size());
  deps_.clear();
  deps_.insert(deps_.end(), off.begin(), off.end());
  dep_idx_at_ = int32_t(deps_.size());
  deps_.insert(deps_.end(), idx.begin(), idx.end());
  dep_joff_at_ = int32_t(deps_.size());
  deps_.insert(deps_.end(), joff.begin(), joff.end());
  dep_jidx_at_ = int32_t(deps_.size());
  deps_.insert(deps_.end(), jidx.begin(), jidx.end());
  upload(d_deps_, d_deps_cap_, deps_);
  if (n > d_done_cap_) {
    OD_CU(cudaStreamSynchronize(s0_));
    cudaFree(d_done_);
    d_done_cap_ = std::max<size_t>(n, tiles4_cap_);
    OD_CU(cudaMalloc(&d_done_, d_done_cap_ * sizeof(unsigned)));
  }
  // every tile has completed every step launched so far (the stream drained)
  if (n > 0) {
    fill_u32<<<64, 256, 0, s0_>>>(d_done_, int(n), unsigned(st_.steps));
    OD_CU(cudaGetLastError());
    ++st_.kernel_launches;
  }
}

void Runtime::rebuild_tables() {
  const double r0 = now_s();
  resident_.clear();
  for (int32_t v = 0; v < K(); ++v)
    if (rank_of_vp(v) == rank_) resident_.push_back(v);
  const int32_t nres = int32_t(resident_.size());
  std::vector<int32_t> slot_of(K(), -1);
  for (int32_t i = 0; i < nres; ++i) slot_of[resident_[i]] = i;

  // tiles, grouped by slot
  std::vector<TileDev> tiles;
  tile_begin_.assign(nres, 0);
  tile_count_.assign(nres, 0);
  for (int32_t i = 0; i < nres; ++i) {
    const Sub& s = subs_[resident_[i]];
    tile_begin_[i] = int32_t(tiles.size());
    for (int32_t ty = 0; ty < s.h(); ty += kTY)
      for (int32_t tx = 0; tx < s.w(); tx += kTX) tiles.push_back(TileDev{i, tx, ty, 0});
    tile_count_[i] = int32_t(tiles.size()) - tile_begin_[i];
  }
  ntiles_ = int32_t(tiles.size());
  upload(d_tiles_, d_tiles_cap_, tiles);
  tiles4_.clear();
  tile4_begin_.assign(nres, 0);
  tile4_count_.assign(nres, 0);
  for (int32_t i = 0; i < nres; ++i) {
    const Sub& s = subs_[resident_[i]];
    tile4_begin_[i] = int32_t(tiles4_.size());
    const int32_t v = resident_[i];
    bool remote[4];
    for (int d = 0; d < 4; ++d) {
      const int32_t n = nbr(v, d);
      remote[d] = n >= 0 && rank_of_vp(n) != rank_;
    }
    const int32_t tw = tile_width(s.w(), s.h()), th = 256 / tw;
    const int32_t lg = tw == 64 ? 5 : tw == 32 ? 4 : tw == 16 ? 3 : 2;
    for (int32_t ty = 0; ty < s.h(); ty += th)
      for (int32_t tx = 0; tx < s.w(); tx += tw) {
        const bool needs = (remote[kLeft] && tx == 0) || (remote[kRight] && tx + tw >= s.w()) ||
                           (remote[kTop] && ty == 0) || (remote[kBottom] && ty + th >= s.h());
        // pad: bit 0 = reads a remote strip, bits 1.. = canonical tile id
        tiles4_.push_back(TileDev{i, tx, ty, (needs ? 1 : 0) | (int32_t(tiles4_.size()) << 1),
                                  tw, th, lg, 0});
      }
    tile4_count_[i] = int32_t(tiles4_.size()) - tile4_begin_[i];
  }
  if (tiles4_.size() > tiles4_cap_) {
    OD_CU(cudaStreamSynchronize(s0_));
    cudaFree(d_tiles4_);
    for (int b = 0; b < 2; ++b) {
      cudaFree(d_tiles4s_[b]);
      if (h_tiles4s_[b]) cudaFreeHost(h_tiles4s_[b]);
    }
    size_t all = 0;
    for (const Sub& sb : subs_) {
      const int32_t tw = tile_width(sb.w(), sb.h()), th = 256 / tw;
      all += size_t((sb.h() + th - 1) / th) * size_t((sb.w() + tw - 1) / tw);
    }
    tiles4_cap_ = std::max<size_t>({tiles4_.size(), all, 16});
    OD_CU(cudaMalloc(&d_tiles4_, tiles4_cap_ * sizeof(TileDev)));
    for (int b = 0; b < 2; ++b) {
      OD_CU(cudaMalloc(&d_tiles4s_[b], tiles4_cap_ * sizeof(TileDev)));
      OD_CU(cudaMallocHost(&h_tiles4s_[b], tiles4_cap_ * sizeof(TileDev)));
      if (!tiles4s_ev_[b]) OD_CU(cudaEventCreateWithFlags(&tiles4s_ev_[b], cudaEventDisableTiming));
    }
  }
  if (!tiles4_.empty())
    OD_CU(cudaMemcpy(d_tiles4_, tiles4_.data(), tiles4_.size() * sizeof(TileDev),
                     cudaMemcpyHostToDevice));
  order_dirty_ = true;
  cur_tiles_ = nullptr;  // (the stream has drained; the next launch refreshes the order)
  oring_pending_ = -1;

  const double r1 = now_s();
  // exchange schedule: per peer, faces in (sender vp, side) order
  jobs_.clear();
  send_off_.assign(world_, 0);
  send_cnt_.assign(world_, 0);
  recv_off_.assign(world_, 0);
  recv_cnt_.assign(world_, 0);
  recv_face_off_.assign(nres, {-1, -1, -1, -1});
  const int64_t per_cell = int64_t(cfg_.nz) * cfg_.fields;
  std::vector<int32_t> rank_of(K());
  for (int32_t v = 0; v < K(); ++v) rank_of[v] = rank_of_vp(v);
  std::vector<FaceXfer> sends, recvs;
  exchange_schedule(subs_, cfg_.decomposition_kind, cfg_.kx, cfg_.ky, rank_of, world_, rank_,
                    per_cell, sends, recvs);
  int64_t soff = 0, roff = 0;
  // receive-side offsets of this rank's strips on each peer (the peer's own
  // schedule, computed here from the same global mapping)
  std::vector<std::vector<int64_t>> remote_off(world_);
  if (p2p_) {
    std::vector<bool> need(world_, false);
    for (const FaceXfer& f : sends) need[f.peer] = true;
    for (int q = 0; q < world_; ++q) {
      if (!need[q]) continue;
      std::vector<FaceXfer> qs, qr;
      exchange_schedule(subs_, cfg_.decomposition_kind, cfg_.kx, cfg_.ky, rank_of, world_, q,
                        per_cell, qs, qr);
      for (const FaceXfer& f : qr)
        if (f.peer == rank_) remote_off[q].push_back(f.offset);
    }
  }
  std::vector<size_t> taken(world_, 0);
  for (const FaceXfer& f : sends) {
    // the receiver's flag of this strip: its chunk f.nbr, face opposite(f.side)
    PackJob pj{slot_of[f.vp], f.side, f.len, f.lenp, f.offset, f.peer,
               world_ + 4 * f.nbr + opposite(f.side), 0};
    if (p2p_) pj.rdst = remote_off[f.peer].at(taken[f.peer]++);
    jobs_.push_back(pj);
    send_cnt_[f.peer] += per_cell * f.lenp;
    soff = f.offset + per_cell * f.lenp;
  }
  for (const FaceXfer& f : recvs) {
    recv_face_off_[slot_of[f.nbr]][opposite(f.side)] = f.offset;
    recv_cnt_[f.peer] += per_cell * f.lenp;
    roff = f.offset + per_cell * f.lenp;
  }
  int64_t so = 0, ro = 0;
  for (int q = 0; q < world_; ++q) {
    send_off_[q] = so;
    recv_off_[q] = ro;
    so += send_cnt_[q];
    ro += recv_cnt_[q];
  }
  if (p2p_) {
    std::vector<int32_t> notify, senders;
    for (int q = 0; q < world_; ++q) {
      if (send_cnt_[q] > 0) notify.push_back(q);
      if (recv_cnt_[q] > 0) senders.push_back(q);
    }
    n_notify_ = int32_t(notify.size());
    n_senders_ = int32_t(senders.size());
    if (n_notify_) OD_CU(cudaMemcpy(d_notify_, notify.data(), notify.size() * 4, cudaMemcpyHostToDevice));
    if (n_senders_) OD_CU(cudaMemcpy(d_senders_, senders.data(), senders.size() * 4, cudaMemcpyHostToDevice));
  }
  if (size_t(soff) > send_cap_) {
    cudaFree(d_send_);
    d_send_ = nullptr;
    send_cap_ = std::max(size_t(soff) * 3 / 2, send_cap_ * 2);
    OD_CU(cudaMalloc(&d_send_, send_cap_ * sizeof(double)));
  }
  if (size_t(roff) > recv_cap_) {
    if (p2p_) throw RuntimeFault("halo receive buffer exceeded its preallocated capacity");
    cudaFree(d_recv_);
    d_recv_ = nullptr;
    recv_cap_ = std::max(size_t(roff) * 3 / 2, recv_cap_ * 2);
    OD_CU(cudaMalloc(&d_recv_, recv_cap_ * sizeof(double)));
  }
  upload(d_jobs_, d_jobs_cap_, jobs_);
  const double r2 = now_s();

  // chunk descriptors for both parities
  for (int par = 0; par < 2; ++par) {
    std::vector<ChunkDev> tab(nres);
    for (int32_t i = 0; i < nres; ++i) {
      const ChunkMem& m = chunks_[resident_[i]];
      ChunkDev& c = tab[i];
      std::memset(&c, 0, sizeof(c));
      c.in = m.u[par];
      c.out = m.u[par ^ 1];
      c.a = m.a;
      c.kstride = m.kstride();
      c.fstride = c.kstride * cfg_.nz;
      c.w = m.sub.w();
      c.h = m.sub.h();
      c.pitch = m.pitch;
      c.x0 = m.sub.x0;
      c.y0 = m.sub.y0;
      c.vp = m.vp;
      c.rmask = 0;
      for (int d = 0; d < 4; ++d) {
        const int32_t n = nbr(m.vp, d);
        if (n < 0) {
          c.face[d] = edge_of(m, d, par);  // zero-flux boundary: the cell itself
        } else if (rank_of_vp(n) == rank_) {
          c.face[d] = edge_of(chunks_[n], opposite(d), par);
        } else {
          const int32_t len = (d == kLeft || d == kRight) ? c.h : c.w;
          c.face[d].p = d_recv_ + par * recv_half_ + recv_face_off_[i][d];
          if (p2p_) c.rmask |= 1 << d;
          c.face[d].lo = d_recv_ + par * recv_half_;
          c.face[d].hi = d_recv_ + par * recv_half_ + int64_t(recv_cap_);
          const int32_t lenp = (len + 1) & ~1;
          c.face[d].fs = int64_t(cfg_.nz) * lenp;
          c.face[d].ks = lenp;
          c.face[d].es = 1;
        }
      }
    }
    if (tma_on_) build_tensor_maps(tab, par, slot_of);
    upload(d_chunks_[par], d_chunks_cap_[par], tab);
  }
  if (!d_trips_ || ns_cols_ < 2 * nres + 1) {
    // per slot (SM-time share ns, executed FP64 ops); last column: the longest
    // in-kernel wait for remote halos (per step)
    ns_cols_ = 2 * std::max(std::max(nres, 1), int(slab_slots_)) + 1;
    cudaFree(d_trips_);
    OD_CU(cudaMalloc(&d_trips_, size_t(ns_cols_) * sizeof(unsigned long long)));
    cudaFree(d_ns_);
    d_ns_ = nullptr;
    ns_rows_ = 0;
  }
  st_.resident_chunks = nres;
  build_step_deps();
  if (trace_on())
    fprintf(stderr, "[od rank %d] rebuild: tiles %.2f ms, exchange %.2f ms, chunk tables %.2f ms\n",
            rank_, (r1 - r0) * 1e3, (r2 - r1) * 1e3, (now_s() - r2) * 1e3);
}

// TMA maps for the full tiles of every resident chunk (parity par): the
// chunk's U^t as a 3-D tensor {w, h, F*nz} (row stride pitch, plane stride
// h*pitch) with a tw x th box and a tw x 1 box, and per top/bottom face the
// tensor its halo row comes from with a tw x 1 box: the neighbour chunk on this
// GPU (row h-1 above, 0 below), the chunk itself (zero-flux edge) or the
// received strip (2-D {lenp, F*nz}).  A chunk without a full tile gets none
// and its tiles keep the cp.async ring.
void Runtime::build_tensor_maps(std::vector<ChunkDev>& tab, int par,
                                const std::vector<int32_t>& slot_of) {
  const int32_t nres = int32_t(tab.size());
  const size_t need = size_t(2) * std::max(nres, 1) * 4;
  if (need > d_tmaps_cap_) {
    OD_CU(cudaStreamSynchronize(s0_));
    cudaFree(d_tmaps_);
    d_tmaps_cap_ = std::max(need, size_t(2) * std::max<size_t>(slab_slots_, 1) * 4);
    OD_CU(cudaMalloc(&d_tmaps_, d_tmaps_cap_ * sizeof(CUtensorMap)));
  }
  std::vector<CUtensorMap> maps(size_t(nres) * 4);
  static const int promo_env = std::getenv("OD_TMA_L2") ? std::atoi(std::getenv("OD_TMA_L2")) : 128;
  const CUtensorMapL2promotion promo = promo_env == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : promo_env == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                       : promo_env == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                          : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  const cuuint64_t planes = cuuint64_t(cfg_.nz) * cfg_.fields;
  auto chunk_map = [&](CUtensorMap* out, const ChunkMem& m, int tw, int rows) {
    const cuuint64_t dims[3] = {cuuint64_t(m.sub.w()), cuuint64_t(m.sub.h()), planes};
    const cuuint64_t strides[2] = {cuuint64_t(m.pitch) * 8, cuuint64_t(m.kstride()) * 8};
    const cuuint32_t box[3] = {cuuint32_t(tw), cuuint32_t(rows), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (encode_tiled_(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, m.u[par], dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      throw RuntimeFault("cuTensorMapEncodeTiled failed for a chunk");
  };
  CUtensorMap* dev = d_tmaps_ + size_t(par) * (d_tmaps_cap_ / 2);
  for (int32_t i = 0; i < nres; ++i) {
    ChunkDev& c = tab[i];
    const ChunkMem& m = chunks_[resident_[i]];
    const int tw = tile_width(c.w, c.h), th = 256 / tw;
    c.tm_main = c.tm_row = nullptr;
    if (c.w < tw || c.h < th || tw < tma_min_width_) continue;  // no full tile / cp.async width
    chunk_map(&maps[size_t(i) * 4 + 0], m, tw, th);
    chunk_map(&maps[size_t(i) * 4 + 1], m, tw, 1);
    for (int side = kTop; side <= kBottom; ++side) {
      CUtensorMap* mp = &maps[size_t(i) * 4 + 2 + (side - kTop)];
      FaceDev& f = c.face[side];
      const int32_t n = nbr(m.vp, side);
      if (n < 0) {  // zero-flux: the chunk's own edge row
        chunk_map(mp, m, tw, 1);
        f.trow = side == kTop ? 0 : c.h - 1;
        f.tkind = 0;
      } else if (rank_of_vp(n) == rank_) {
        const ChunkMem& nm = chunks_[n];
        chunk_map(mp, nm, tw, 1);
        f.trow = side == kTop ? nm.sub.h() - 1 : 0;
        f.tkind = 0;
      } else {  // received strip [f][k][e], e along x
        const cuuint64_t lenp = cuuint64_t((c.w + 1) & ~1);
        const cuuint64_t dims[2] = {cuuint64_t(c.w), planes};
        const cuuint64_t strides[1] = {lenp * 8};
        const cuuint32_t box[2] = {cuuint32_t(tw), 1};
        const cuuint32_t es[2] = {1, 1};
        if (encode_tiled_(mp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(f.p), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          throw RuntimeFault("cuTensorMapEncodeTiled failed for a received strip");
        f.trow = 0;
        f.tkind = 1;
      }
      f.tm = dev + size_t(i) * 4 + 2 + (side - kTop);
    }
    c.tm_main = dev + size_t(i) * 4 + 0;
    c.tm_row = dev + size_t(i) * 4 + 1;
  }
  (void)slot_of;
  if (nres > 0)
    OD_CU(cudaMemcpy(dev, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
}

// Worst case for this rank: every face of every chunk slot borders another GPU.
void Runtime::alloc_comm_buffers() {
  size_t per = 0;
  for (const Sub& sb : subs_)
    per = std::max<size_t>(per, size_t(2 * (((sb.w() + 1) & ~1) + ((sb.h() + 1) & ~1))));
  size_t resident = 0;
  for (int32_t v = 0; v < K(); ++v) resident += rank_of_vp(v) == rank_;
  const size_t slots = std::max<size_t>(slab_slots_, resident);
  send_cap_ = recv_cap_ = per * size_t(cfg_.nz) * cfg_.fields * slots;
  OD_CU(cudaMalloc(&d_send_, send_cap_ * sizeof(double)));
  recv_half_ = p2p_ ? int64_t(recv_cap_) : 0;
  OD_CU(cudaMalloc(&d_recv_, (p2p_ ? 2 : 1) * recv_cap_ * sizeof(double)));
}

// Map every peer's receive buffer and flag array into this process (CUDA IPC;
// handles all-gathered over the NCCL communicator).
void Runtime::setup_p2p() {
  OD_CU(cudaMalloc(&d_flags_, sizeof(unsigned long long) * (world_ + 4 * size_t(K()))));
  OD_CU(cudaMemset(d_flags_, 0, sizeof(unsigned long long) * (world_ + 4 * size_t(K()))));
  OD_CU(cudaMalloc(&d_jcnt1_, 4 * size_t(K()) * sizeof(unsigned)));
  OD_CU(cudaMalloc(&d_pack_counter_, sizeof(unsigned int)));
  OD_CU(cudaMemset(d_pack_counter_, 0, sizeof(unsigned int)));
  // senders address a peer's parity half as peer_base + par * half, so every
  // rank's half must have the same size: the largest rank's (resident chunk
  // counts, hence worst-case capacities, differ between ranks)
  {
    int64_t* d_cap = nullptr;
    OD_CU(cudaMalloc(&d_cap, sizeof(int64_t) * (world_ + 1)));
    const int64_t cap = int64_t(recv_cap_);
    OD_CU(cudaMemcpy(d_cap, &cap, sizeof(int64_t), cudaMemcpyHostToDevice));
    OD_NC(odb::nccl().AllGather(d_cap, d_cap + 1, 1, ncclInt64, comm_, s0_));
    std::vector<int64_t> caps(world_);
    OD_CU(cudaMemcpyAsync(caps.data(), d_cap + 1, sizeof(int64_t) * world_,
                          cudaMemcpyDeviceToHost, s0_));
    OD_CU(cudaStreamSynchronize(s0_));
    cudaFree(d_cap);
    const size_t top = size_t(*std::max_element(caps.begin(), caps.end()));
    if (top > recv_cap_) {
      cudaFree(d_recv_);
      recv_cap_ = top;
      OD_CU(cudaMalloc(&d_recv_, 2 * recv_cap_ * sizeof(double)));
    }
    recv_half_ = int64_t(recv_cap_);
  }
  // [recv buffer, flags, chunk slab (migration pulls; zeroed if no slab)]
  cudaIpcMemHandle_t mine[3];
  std::memset(mine, 0, sizeof(mine));
  OD_CU(cudaIpcGetMemHandle(&mine[0], d_recv_));
  OD_CU(cudaIpcGetMemHandle(&mine[1], d_flags_));
  if (slab_) OD_CU(cudaIpcGetMemHandle(&mine[2], slab_));
  const size_t hb = sizeof(mine);
  uint8_t* d_h = nullptr;
  OD_CU(cudaMalloc(&d_h, hb * (world_ + 1)));
  OD_CU(cudaMemcpy(d_h, mine, hb, cudaMemcpyHostToDevice));
  OD_CU(cudaDeviceSynchronize());
  OD_NC(odb::nccl().AllGather(d_h, d_h + hb, hb, ncclUint8, comm_, s0_));
  std::vector<cudaIpcMemHandle_t> all(3 * world_);
  OD_CU(cudaMemcpyAsync(all.data(), d_h + hb, hb * world_, cudaMemcpyDeviceToHost, s0_));
  OD_CU(cudaStreamSynchronize(s0_));
  cudaFree(d_h);
  peer_recv_.assign(world_, nullptr);
  peer_flags_.assign(world_, nullptr);
  peer_slab_.assign(world_, nullptr);
  const cudaIpcMemHandle_t zero{};
  peer_slabs_ok_ = true;
  for (int q = 0; q < world_; ++q) {
    if (q == rank_) {
      peer_recv_[q] = d_recv_;
      peer_flags_[q] = d_flags_;
      peer_slab_[q] = slab_;
      peer_slabs_ok_ = peer_slabs_ok_ && slab_ != nullptr;
      continue;
    }
    void* p = nullptr;
    OD_CU(cudaIpcOpenMemHandle(&p, all[3 * q], cudaIpcMemLazyEnablePeerAccess));
    peer_recv_[q] = static_cast<double*>(p);
    OD_CU(cudaIpcOpenMemHandle(&p, all[3 * q + 1], cudaIpcMemLazyEnablePeerAccess));
    peer_flags_[q] = static_cast<unsigned long long*>(p);
    if (std::memcmp(&all[3 * q + 2], &zero, sizeof(zero)) != 0) {
      OD_CU(cudaIpcOpenMemHandle(&p, all[3 * q + 2], cudaIpcMemLazyEnablePeerAccess));
      peer_slab_[q] = static_cast<double*>(p);
    } else {
      peer_slabs_ok_ = false;
    }
  }
  OD_CU(cudaMalloc(&d_peer_base_, sizeof(double*) * world_));
  OD_CU(cudaMemcpy(d_peer_base_, peer_recv_.data(), sizeof(double*) * world_,
                   cudaMemcpyHostToDevice));
  OD_CU(cudaMalloc(&d_peer_flags_, sizeof(unsigned long long*) * world_));
  OD_CU(cudaMemcpy(d_peer_flags_, peer_flags_.data(), sizeof(unsigned long long*) * world_,
                   cudaMemcpyHostToDevice));
  OD_CU(cudaMalloc(&d_notify_, sizeof(int32_t) * world_));
  OD_CU(cudaMalloc(&d_senders_, sizeof(int32_t) * world_));
}

// ------------------------------------------------------------------- steps --

int Runtime::new_event() {
  if (ev_used_ == int(events_.size())) {
    cudaEvent_t e;
    OD_CU(cudaEventCreate(&e));
    events_.push_back(e);
  }
  return ev_used_++;
}

void Runtime::begin_window(bool allow_overlap) {
  window_.clear();
  ev_used_ = 0;
  ns_used_ = 0;
  win_overlap_ = overlap_ && allow_overlap && cfg_.overlap != 0 && !d_tl_ &&
                 (cfg_.measure == OD_MEASURE_TIMER || cfg_.measure == OD_MEASURE_TIMER_RAW);
  if (oring_pending_ >= 0) {
    // the stream has drained (collect): the last mapped order becomes the device list
    const int b = tiles4s_cur_ ^ 1;
    const size_t n = tiles4_.size();
    OD_CU(cudaEventSynchronize(tiles4s_ev_[b]));
    std::memcpy(h_tiles4s_[b], h_oring_[oring_pending_], n * sizeof(TileDev));
    OD_CU(cudaMemcpyAsync(d_tiles4s_[b], h_tiles4s_[b], n * sizeof(TileDev),
                          cudaMemcpyHostToDevice, s0_));
    OD_CU(cudaEventRecord(tiles4s_ev_[b], s0_));
    tiles4s_cur_ = b;
    cur_tiles_ = d_tiles4s_[b];
    oring_pending_ = -1;
  }
  if (win_overlap_) {
    const int32_t S = std::max(cfg_.async_steps + cfg_.sync_steps, 1);
    if (int(h_oring_.size()) < S || oring_cap_ < tiles4_cap_) {
      OD_CU(cudaStreamSynchronize(s0_));
      for (TileDev* h : h_oring_) cudaFreeHost(h);
      h_oring_.clear();
      d_oring_.clear();
      oring_cap_ = tiles4_cap_;
      for (int32_t i = 0; i < S; ++i) {
        TileDev* h = nullptr;
        TileDev* d = nullptr;
        OD_CU(cudaHostAlloc(reinterpret_cast<void**>(&h), std::max<size_t>(oring_cap_, 1) * sizeof(TileDev),
                            cudaHostAllocMapped));
        OD_CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0));
        h_oring_.push_back(h);
        d_oring_.push_back(d);
      }
    }
    if (win_cap_ < S) {
      OD_CU(cudaStreamSynchronize(s0_));
      cudaFree(d_stepend_);
      cudaFree(d_pcnt_);
      cudaFree(d_jcnt_);
      win_cap_ = S;
      OD_CU(cudaMalloc(&d_jcnt_, size_t(S) * 4 * size_t(K()) * sizeof(unsigned)));
      OD_CU(cudaMalloc(&d_stepend_, size_t(2 * S) * sizeof(unsigned long long)));
      OD_CU(cudaMalloc(&d_pcnt_, size_t(4 * S) * sizeof(unsigned)));
    }
    OD_CU(cudaMemsetAsync(d_stepend_, 0, size_t(2 * win_cap_) * sizeof(unsigned long long), s0_));
    OD_CU(cudaMemsetAsync(d_pcnt_, 0, size_t(4 * win_cap_) * sizeof(unsigned), s0_));
    OD_CU(cudaMemsetAsync(d_jcnt_, 0, size_t(win_cap_) * 4 * size_t(K()) * sizeof(unsigned), s0_));
    // every tile is current with every step launched so far (earlier steps may
    // have run without the per-tile stamps)
    if (!tiles4_.empty()) {
      fill_u32<<<64, 256, 0, s0_>>>(d_done_, int(tiles4_.size()), unsigned(st_.steps));
      OD_CU(cudaGetLastError());
      ++st_.kernel_launches;
    }
    // measured rows zeroed up front: no per-step memset between the kernels
    if (ns_cols_ > 0) {
      if (ns_rows_ < S) {
        OD_CU(cudaStreamSynchronize(s0_));
        cudaFree(d_ns_);
        ns_rows_ = S;
        OD_CU(cudaMalloc(&d_ns_, size_t(ns_rows_) * ns_cols_ * sizeof(unsigned long long)));
      }
      OD_CU(cudaMemsetAsync(d_ns_, 0, size_t(ns_rows_) * ns_cols_ * sizeof(unsigned long long), s0_));
    }
  }
  prof_j_.clear();
  prof_p_.clear();
  prof_f_.clear();
  prof_pack_.clear();
  prof_x_.clear();
}

void Runtime::launch_step(int32_t mode, int32_t epoch_step, bool host_io,
                          const double* host_field, int staged_slot) {
  const auto t0 = std::chrono::steady_clock::now();
  StepRec r;
  r.mode = mode;
  r.epoch_step = epoch_step;
  // per-step device slots (step stamps, pack counters, mapped field buffers)
  // are indexed by the step's position in the window, never by the label
  const int32_t pos = int32_t(window_.size());
  r.pos = pos;
  r.gstep = st_.steps;
  r.slot_vps = resident_;
  const int par = parity_;
  const int32_t nres = int32_t(resident_.size());
  const bool timer = host_io || (mode == kSync && (cfg_.measure == OD_MEASURE_TIMER ||
                                                    cfg_.measure == OD_MEASURE_TIMER_RAW ||
                                                    cfg_.measure == OD_MEASURE_OPS));
  // overlapped step: launched with programmatic dependent launch right behind
  // the previous step kernel; no stream operation may sit between them
  r.ovl = win_overlap_ && pos < win_cap_ &&
          (!host_io || staged_slot >= 0 || int32_t(d_ring_.size()) > pos) &&
          !tiles4_.empty() && (mode == kAsync || timer);
  r.ovl_chained = r.ovl && !window_.empty() && window_.back().ovl;
  // a refreshed order inside a chain travels in mapped memory (no stream op)
  if (r.ovl && order_dirty_) refresh_tile_order(r.ovl_chained ? pos : -1);
  if (!r.ovl) {
    r.ev_begin = new_event();
    OD_CU(cudaEventRecord(events_[r.ev_begin], s0_));
  } else if (!r.ovl_chained) {
    stamp_time<<<1, 1, 0, s0_>>>(d_stepend_ + 2 * pos);  // start of a chain
    ++st_.kernel_launches;
  }
  tl_mark(0);

  const double* cfield = d_cbase_;
  int32_t shift = shift_ % cfg_.ny;
  // host-facing steps: the step's load field comes from the caller's host
  // buffer (or, without one, the runtime's own shifted field, which the
  // reference keeps on the host: engine.hpp:337-342)
  const double* hsrc = host_field ? host_field : field_.c.data();
  if (host_io && r.ovl && staged_slot >= 0) {
    // the caller's field for this step was staged while the previous step ran
    cfield = d_ring_[staged_slot];
    shift = 0;
  } else if (host_io && r.ovl) {
    // overlapped: the step kernel reads this step's mapped pinned copy over the
    // host link (8 B per column per step, no copy operation between the kernels)
    std::memcpy(h_ring_[pos], hsrc, field_.c.size() * sizeof(double));
    cfield = d_ring_[pos];
    shift = 0;
  } else if (host_io) {
    const int b = cstage_cur_ ^= 1;
    OD_CU(cudaEventSynchronize(cstage_ev_[b]));  // the copy two steps ago has left it
    std::memcpy(h_cstage_[b], hsrc, field_.c.size() * sizeof(double));
    OD_CU(cudaMemcpyAsync(d_cstage_[b], h_cstage_[b], field_.c.size() * sizeof(double),
                          cudaMemcpyHostToDevice, s0_));
    OD_CU(cudaEventRecord(cstage_ev_[b], s0_));
    cfield = d_cstage_[b];
    shift = 0;
  }
  unsigned long long* ns = nullptr;
  if (timer) {
    if (ns_used_ == ns_rows_) {
      // grow the counter matrix (rare: first use or a longer window)
      const int rows = std::max(ns_rows_ * 2, cfg_.sync_steps + 1);
      unsigned long long* nd = nullptr;
      OD_CU(cudaStreamSynchronize(s0_));
      OD_CU(cudaMalloc(&nd, size_t(rows) * ns_cols_ * sizeof(unsigned long long)));
      if (d_ns_) {
        OD_CU(cudaMemcpy(nd, d_ns_, size_t(ns_rows_) * ns_cols_ * sizeof(unsigned long long),
                         cudaMemcpyDeviceToDevice));
        cudaFree(d_ns_);
      }
      d_ns_ = nd;
      ns_rows_ = rows;
    }
    r.ns_row = ns_used_++;
    ns = d_ns_ + size_t(r.ns_row) * ns_cols_;
    if (!r.ovl)  // overlapped windows zero their rows up front
      OD_CU(cudaMemsetAsync(ns, 0, size_t(ns_cols_) * sizeof(unsigned long long), s0_));
  }

  // boundaries of chunks that border another GPU
  const bool fused = cfg_.overlap != 0 && !tiles4_.empty() && (mode == kAsync || timer);
  const bool fused_pack = p2p_ && pack_ctas_ > 0 && fused;
  if (p2p_ && (!jobs_.empty() || n_senders_ > 0)) {
    // pack straight into the neighbours' receive buffers over NVLink, publish
    // the step, then wait for the neighbours' strips of this step
    int e0 = -1, e1 = -1, e2 = -1;
    const bool prof_x = profiling_ && !r.ovl;
    if (prof_x) {
      e0 = new_event();
      OD_CU(cudaEventRecord(events_[e0], s0_));
    }
    const unsigned long long stamp = (unsigned long long)(st_.steps + 1);
    if (!jobs_.empty() && fused_pack) {
      // packed by the persistent kernel's first CTAs (pack_units)
      for (int q = 0; q < world_; ++q) st_.halo_bytes_sent += send_cnt_[q] * int64_t(sizeof(double));
    } else if (!jobs_.empty()) {
      pack_faces_p2p<<<dim3(unsigned(jobs_.size()), unsigned(cfg_.fields)), 256, 0, s0_>>>(
          d_chunks_[par], d_jobs_, d_peer_base_, recv_half_, par, cfg_.nz, d_pack_counter_,
          d_peer_flags_, d_notify_, n_notify_, rank_, stamp);
      OD_CU(cudaGetLastError());
      ++st_.kernel_launches;
      for (int q = 0; q < world_; ++q) st_.halo_bytes_sent += send_cnt_[q] * int64_t(sizeof(double));
    }
    if (prof_x) {
      e1 = new_event();
      OD_CU(cudaEventRecord(events_[e1], s0_));
    }
    // the fused step kernels wait inside, per tile that needs a remote strip
    // (pre-rolling its physics); the separate kernels wait here
    const bool in_kernel = fused;
    if (n_senders_ > 0 && !in_kernel) {
      wait_halo<<<1, 32, 0, s0_>>>(d_flags_, d_senders_, n_senders_, stamp,
                                   20ull * 1000 * 1000 * 1000);
      OD_CU(cudaGetLastError());
      ++st_.kernel_launches;
    }
    if (prof_x) {
      e2 = new_event();
      OD_CU(cudaEventRecord(events_[e2], s0_));
      prof_pack_.push_back({e0, e1});
      prof_x_.push_back({e1, e2});
    }
  } else if (!jobs_.empty() || (world_ > 1 && std::any_of(recv_cnt_.begin(), recv_cnt_.end(),
                                                          [](int64_t c) { return c > 0; }))) {
    int e0 = -1, e1 = -1, e2 = -1;
    if (profiling_) {
      e0 = new_event();
      OD_CU(cudaEventRecord(events_[e0], s0_));
    }
    if (!jobs_.empty()) {
      pack_faces<<<dim3(unsigned(jobs_.size()), unsigned(cfg_.fields)), 256, 0, s0_>>>(
          d_chunks_[par], d_jobs_, d_send_, cfg_.nz);
      OD_CU(cudaGetLastError());
      ++st_.kernel_launches;
    }
    if (profiling_) {
      e1 = new_event();
      OD_CU(cudaEventRecord(events_[e1], s0_));
    }
    OD_NC(odb::nccl().GroupStart());
    for (int q = 0; q < world_; ++q) {
      if (q == rank_) continue;
      if (send_cnt_[q] > 0)
        OD_NC(odb::nccl().Send(d_send_ + send_off_[q], size_t(send_cnt_[q]), ncclFloat64, q, comm_, s0_));
      if (recv_cnt_[q] > 0)
        OD_NC(odb::nccl().Recv(d_recv_ + recv_off_[q], size_t(recv_cnt_[q]), ncclFloat64, q, comm_, s0_));
      st_.halo_bytes_sent += send_cnt_[q] * int64_t(sizeof(double));
    }
    OD_NC(odb::nccl().GroupEnd());
    if (profiling_) {
      e2 = new_event();
      OD_CU(cudaEventRecord(events_[e2], s0_));
      prof_pack_.push_back({e0, e1});
      prof_x_.push_back({e1, e2});
    }
  }

  tl_mark(1);
  const bool slog = d_slog_ && timer && long(st_.steps) == slog_step_;
  if (slog) slog_arm(true);
  const dim3 blk(kTX, kTY);
  if (timer && !r.ovl) {
    r.kev0 = new_event();
    OD_CU(cudaEventRecord(events_[r.kev0], s0_));
  }
  if (fused) {
    if (order_dirty_) refresh_tile_order();
    if (!cur_tiles_) cur_tiles_ = d_tiles4s_[tiles4s_cur_];
    int e0 = -1, e1 = -1;
    const bool prof_f = profiling_ && !r.ovl;
    if (prof_f) {
      e0 = new_event();
      OD_CU(cudaEventRecord(events_[e0], s0_));
    }
    if (!r.ovl) OD_CU(cudaMemsetAsync(d_counter_, 0, 3 * sizeof(unsigned int), s0_));
    tl_mark(2);
    const int nt = int(tiles4_.size());
    PackArgs pk{};
    if (fused_pack && !jobs_.empty()) {
      // pack-only CTAs ahead of the tiles
      pk.jobs = d_jobs_;
      pk.njobs = int32_t(jobs_.size());
      pk.ctas = std::min(pack_ctas_, int(pk.njobs) * cfg_.fields);
      pk.peer_base = d_peer_base_;
      pk.half_elems = recv_half_;
      pk.par = par;
      pk.n_notify = n_notify_;
      pk.my_rank = rank_;
      pk.first = 0;
      pk.counters = r.ovl ? d_pcnt_ + 4 * pos : d_counter_ + 1;
      pk.jcnt = r.ovl ? d_jcnt_ + size_t(pos) * 4 * size_t(K()) : d_jcnt1_;
      if (!r.ovl)
        OD_CU(cudaMemsetAsync(pk.jcnt, 0, jobs_.size() * sizeof(unsigned), s0_));
      pk.peer_flags = d_peer_flags_;
      pk.notify = d_notify_;
    }
    const int32_t face_base = world_;  // per-face flags follow the per-sender ones
    const unsigned long long stamp = (unsigned long long)(st_.steps + 1);
    StepDeps sd{};
    if (r.ovl) {
      sd.off = d_deps_;
      sd.idx = d_deps_ + dep_idx_at_;
      sd.joff = d_deps_ + dep_joff_at_;
      sd.jidx = d_deps_ + dep_jidx_at_;
      sd.done = d_done_;
      sd.end_ns = d_stepend_ + 2 * pos + 1;
      sd.step = unsigned(st_.steps);
      sd.on = 1;
      if (host_io && nres > 0) {
        sd.tile_cnt = d_pcnt_ + 4 * pos + 2;
        sd.ntiles = nt;
        sd.res_words = 2 * nres;
        sd.res_dst = d_loads_dst_;
      }
    }
    // overlapped steps: programmatic dependent launch, so this grid starts
    // while the previous step's last tiles drain (tiles wait on per-tile stamps)
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(nt + pk.ctas));
    lc.blockDim = dim3(32, kRowWarps);
    lc.stream = s0_;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = la;
    lc.numAttrs = r.ovl ? 1 : 0;
    const TileDev* tl4 = cur_tiles_;
    const ChunkDev* chk = d_chunks_[par];
    unsigned long long* nsp = timer ? ns : nullptr;
    unsigned long long* waitp = timer ? ns + (ns_cols_ - 1) : (r.ovl ? nullptr : tl_wait());
    if (use_ws()) {
      // warp-specialised tiles (column_step_ws): physics and Jacobi warps
      lc.blockDim = dim3(32, 2 * kRowWarps);
      // a grid that fits the GPU one tile per SM is spread one per SM: unused
      // dynamic shared memory caps the kernel at one CTA per SM, so no two
      // tiles' serial physics chains share an SM's FP64 pipe (the block
      // scheduler packs small grids onto fewer SMs otherwise; 128 heavy tiles:
      // 1.95 -> 1.71 ms per step).  OD_WS_SPREAD=0 turns it off.
      if (ws_spread_ && nt + pk.ctas <= sms_) lc.dynamicSmemBytes = kWsSpreadSmem;
      if (timer)
        OD_CU(cudaLaunchKernelEx(&lc, column_step_ws<kFusedPrefetch, true, kWsMinBlocks>, chk,
                                 tl4, cfg_.nz, cfg_.fields, cfield, cfg_.nx, cfg_.ny, shift,
                                 cfg_.n_inner, nsp, (const unsigned long long*)d_flags_,
                                 face_base, stamp, waitp, pk, sd));
      else
        OD_CU(cudaLaunchKernelEx(&lc, column_step_ws<kFusedPrefetch, false, kWsMinBlocks>, chk,
                                 tl4, cfg_.nz, cfg_.fields, cfield, cfg_.nx, cfg_.ny, shift,
                                 cfg_.n_inner, nsp, (const unsigned long long*)d_flags_,
                                 face_base, stamp, waitp, pk, sd));
      last_kernel_ = OD_KERNEL_STEP_WS;
    } else {
      // interleaved tiles (column_step_grid)
      if (timer)
        OD_CU(cudaLaunchKernelEx(&lc, column_step_grid<kFusedPrefetch, true, kGridMinBlocks>,
                                 chk, tl4, cfg_.nz, cfg_.fields, cfield, cfg_.nx, cfg_.ny, shift,
                                 cfg_.n_inner, nsp, (const unsigned long long*)d_flags_,
                                 face_base, stamp, waitp, pk, sd));
      else
        OD_CU(cudaLaunchKernelEx(&lc, column_step_grid<kFusedPrefetch, false, kGridMinBlocks>,
                                 chk, tl4, cfg_.nz, cfg_.fields, cfield, cfg_.nx, cfg_.ny, shift,
                                 cfg_.n_inner, nsp, (const unsigned long long*)d_flags_,
                                 face_base, stamp, waitp, pk, sd));
      last_kernel_ = OD_KERNEL_STEP_GRID;
    }
    OD_CU(cudaGetLastError());
    if (prof_f) {
      e1 = new_event();
      OD_CU(cudaEventRecord(events_[e1], s0_));
      prof_f_.push_back({e0, e1});
    }
    st_.kernel_launches += 1;
    st_.fused_launches += 1;
  } else if (mode == kAsync || timer) {
    int e0 = -1, e1 = -1, e2 = -1;
    if (profiling_) {
      e0 = new_event();
      OD_CU(cudaEventRecord(events_[e0], s0_));
    }
    if (ntiles_ > 0) {
      if (timer)
        jacobi_step<kTX, kTY, kPrefetch, true><<<dim3(ntiles_, cfg_.fields), blk, 0, s0_>>>(
            d_chunks_[par], d_tiles_, cfg_.nz, ns);
      else
        jacobi_step<kTX, kTY, kPrefetch, false><<<dim3(ntiles_, cfg_.fields), blk, 0, s0_>>>(
            d_chunks_[par], d_tiles_, cfg_.nz, nullptr);
      OD_CU(cudaGetLastError());
      if (profiling_) {
        e1 = new_event();
        OD_CU(cudaEventRecord(events_[e1], s0_));
      }
      if (timer)
        physics_step<kTX, kTY, true, false><<<ntiles_, blk, 0, s0_>>>(
            d_chunks_[par], d_tiles_, cfield, cfg_.nx, cfg_.ny, shift, cfg_.nz, cfg_.n_inner, ns,
            nullptr);
      else
        physics_step<kTX, kTY, false, false><<<ntiles_, blk, 0, s0_>>>(
            d_chunks_[par], d_tiles_, cfield, cfg_.nx, cfg_.ny, shift, cfg_.nz, cfg_.n_inner,
            nullptr, nullptr);
      OD_CU(cudaGetLastError());
      st_.kernel_launches += 2;
      st_.jacobi_launches += 1;
      st_.physics_launches += 1;
      last_kernel_ = OD_KERNEL_SEPARATE;
      if (profiling_) {
        e2 = new_event();
        OD_CU(cudaEventRecord(events_[e2], s0_));
        prof_j_.push_back({e0, e1});
        prof_p_.push_back({e1, e2});
      }
    }
  } else {
    // paper protocol: serialised per-chunk launches with
    // an event pair around each chunk's Jacobi + physics
    r.chunk_ev0 = ev_used_;
    for (int32_t i = 0; i < nres; ++i) {
      const int eb = new_event(), ee = new_event();
      OD_CU(cudaEventRecord(events_[eb], s0_));
      if (cfg_.overlap != 0) {
        // the chunk's tiles through the interleaved tile kernel (no overlap, no pack)
        column_step_grid<kFusedPrefetch, false, kGridMinBlocks>
            <<<tile4_count_[i], dim3(32, kRowWarps), 0, s0_>>>(
                d_chunks_[par], d_tiles4_ + tile4_begin_[i], cfg_.nz, cfg_.fields, cfield,
                cfg_.nx, cfg_.ny, shift, cfg_.n_inner, nullptr, d_flags_, world_, 0ull,
                nullptr, PackArgs{}, StepDeps{});
        st_.kernel_launches += 1;
        st_.fused_launches += 1;
      } else {
        jacobi_step<kTX, kTY, kPrefetch, false>
            <<<dim3(tile_count_[i], cfg_.fields), blk, 0, s0_>>>(
                d_chunks_[par], d_tiles_ + tile_begin_[i], cfg_.nz, nullptr);
        physics_step<kTX, kTY, false, false><<<tile_count_[i], blk, 0, s0_>>>(
            d_chunks_[par], d_tiles_ + tile_begin_[i], cfield, cfg_.nx, cfg_.ny, shift, cfg_.nz,
            cfg_.n_inner, nullptr, nullptr);
        st_.kernel_launches += 2;
        st_.jacobi_launches += 1;
        st_.physics_launches += 1;
      }
      OD_CU(cudaGetLastError());
      OD_CU(cudaEventRecord(events_[ee], s0_));
    }
  }
  if (timer && !r.ovl) {
    r.kev1 = new_event();
    OD_CU(cudaEventRecord(events_[r.kev1], s0_));
  }
  tl_mark(3);
  if (slog) slog_arm(false);
  if (timer && ns && tl_wait()) copy_u64<<<1, 1, 0, s0_>>>(tl_wait(), ns + (ns_cols_ - 1));
  if (d_tl_ && tl_n_ < tl_cap_) ++tl_n_;
  if (host_io && nres > 0 && !r.ovl) {
    // the step's per-chunk device times back to the host (overlapped steps:
    // written by the kernel's last CTA into the mapped row)
    OD_CU(cudaMemcpyAsync(h_loads_dst_, ns, size_t(2 * nres) * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s0_));
  }
  if (!r.ovl) {
    r.ev_end = new_event();
    OD_CU(cudaEventRecord(events_[r.ev_end], s0_));
  }
  parity_ ^= 1;
  ++st_.steps;
  r.host_launch_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  window_.push_back(std::move(r));
}

static double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  OD_CU(cudaEventElapsedTime(&ms, a, b));
  return double(ms) * 1e-3;
}

void Runtime::collect(std::vector<double>& walls, std::vector<double>& samples) {
  OD_CU(cudaStreamSynchronize(s0_));
  if (trace_on()) tr_drained_ = now_s();
  const int32_t S = int32_t(window_.size());
  const int32_t Kv = K();
  std::vector<unsigned long long> ns;
  if (ns_used_ > 0) {
    ns.resize(size_t(ns_used_) * ns_cols_);
    OD_CU(cudaMemcpy(ns.data(), d_ns_, ns.size() * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost));
  }
  // overlapped steps: device stamps (chain start, last tile end per step)
  std::vector<unsigned long long> stamps;
  if (std::any_of(window_.begin(), window_.end(), [](const StepRec& r) { return r.ovl; })) {
    stamps.resize(size_t(2) * win_cap_);
    OD_CU(cudaMemcpy(stamps.data(), d_stepend_, stamps.size() * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost));
  }
  // local rows: [S*K samples | S walls]
  const size_t row = size_t(S) * Kv + S;
  std::vector<double> local(row, 0.0);
  for (int32_t s = 0; s < S; ++s) {
    const StepRec& r = window_[s];
    if (r.ovl) {
      const int es = r.pos;
      const unsigned long long end = stamps[2 * es + 1];
      const unsigned long long start =
          r.ovl_chained && es > 0 ? stamps[2 * (es - 1) + 1] : stamps[2 * es];
      const double w = end > start ? double(end - start) * 1e-9 : 0.0;
      local[size_t(S) * Kv + s] = w;
      if (profiling_) {
        st_.fused_ms += w * 1e3;  // the step's kernel time, overlap included
        st_.fused_timed += 1;
      }
    } else {
      local[size_t(S) * Kv + s] = elapsed_s(events_[r.ev_begin], events_[r.ev_end]);
    }
    // TIMER: the chunk's processor-sharing SM time (sum over its tiles of
    // integral dt / resident CTAs on the tile's SM) divided by the SM count, in
    // seconds of the whole GPU.  A GPU's samples sum to its mean SM busy time;
    // CTAs spinning on a peer's halo are not resident in a tile, so time a GPU
    // idles for its neighbours is charged to nobody.  TIMER_RAW: the same shares
    // in SM-seconds.  OPS: the event-timed kernel time minus the longest
    // in-kernel halo wait, apportioned by the FP64 instructions each chunk
    // executed (ignores the Jacobi's HBM time).
    const bool by_ops = cfg_.measure == OD_MEASURE_OPS && r.kev0 >= 0;
    double sum = 0, kt = 0;
    if (r.ns_row >= 0 && r.mode == kSync && by_ops) {
      for (size_t j = 0; j < r.slot_vps.size(); ++j)
        sum += double(ns[size_t(r.ns_row) * ns_cols_ + 2 * j + 1]);
      const double wait = double(ns[size_t(r.ns_row) * ns_cols_ + (ns_cols_ - 1)]) * 1e-9;
      kt = std::max(0.0, elapsed_s(events_[r.kev0], events_[r.kev1]) - wait);
    }
    for (size_t i = 0; i < r.slot_vps.size(); ++i) {
      double v;
      if (r.ns_row >= 0 && r.mode == kSync) {
        v = double(ns[size_t(r.ns_row) * ns_cols_ + 2 * i]) * 1e-9;
        if (cfg_.measure == OD_MEASURE_TIMER) v /= double(sms_);
        if (by_ops)
          v = sum > 0 ? double(ns[size_t(r.ns_row) * ns_cols_ + 2 * i + 1]) / sum * kt : 0.0;
      }
      else if (r.mode == kSync && r.chunk_ev0 >= 0)
        v = elapsed_s(events_[r.chunk_ev0 + 2 * i], events_[r.chunk_ev0 + 2 * i + 1]);
      else
        v = r.host_launch_s;  // launch_only_sample: only the launch is visible
      local[size_t(s) * Kv + r.slot_vps[i]] = v;
    }
  }
  for (auto& p : prof_j_) st_.jacobi_ms += elapsed_s(events_[p.first], events_[p.second]) * 1e3;
  for (auto& p : prof_p_) st_.physics_ms += elapsed_s(events_[p.first], events_[p.second]) * 1e3;
  for (auto& p : prof_f_) st_.fused_ms += elapsed_s(events_[p.first], events_[p.second]) * 1e3;
  st_.fused_timed += int64_t(prof_f_.size());
  st_.jacobi_timed += int64_t(prof_j_.size());
  st_.physics_timed += int64_t(prof_p_.size());
  for (auto& p : prof_pack_) st_.pack_ms += elapsed_s(events_[p.first], events_[p.second]) * 1e3;
  for (auto& p : prof_x_) st_.exchange_ms += elapsed_s(events_[p.first], events_[p.second]) * 1e3;

  walls.assign(S, 0.0);
  samples.assign(size_t(S) * Kv, 0.0);
  auto keep_walls = [&] {
    for (int32_t s = 0; s < S; ++s) {
      const size_t g = size_t(window_[s].gstep);
      if (step_wall_.size() <= g) step_wall_.resize(g + 1, std::nan(""));
      step_wall_[g] = walls[s];
    }
  };
  if (world_ == 1) {
    std::copy(local.begin(), local.begin() + size_t(S) * Kv, samples.begin());
    for (int32_t s = 0; s < S; ++s) walls[s] = local[size_t(S) * Kv + s];
    keep_walls();
    return;
  }
  const size_t need = row * (world_ + 1);
  if (need > gather_cap_) {
    cudaFree(d_gather_);
    d_gather_ = nullptr;
    gather_cap_ = need;
    OD_CU(cudaMalloc(&d_gather_, gather_cap_ * sizeof(double)));
  }
  OD_CU(cudaMemcpy(d_gather_, local.data(), row * sizeof(double), cudaMemcpyHostToDevice));
  OD_NC(odb::nccl().AllGather(d_gather_, d_gather_ + row, row, ncclFloat64, comm_, s0_));
  std::vector<double> all(row * world_);
  OD_CU(cudaMemcpyAsync(all.data(), d_gather_ + row, all.size() * sizeof(double),
                        cudaMemcpyDeviceToHost, s0_));
  OD_CU(cudaStreamSynchronize(s0_));
  // values are taken from the owning rank (selection, no arithmetic)
  for (int32_t s = 0; s < S; ++s) {
    double mx = 0;
    for (int q = 0; q < world_; ++q) mx = std::max(mx, all[q * row + size_t(S) * Kv + s]);
    walls[s] = mx;
    for (int32_t v = 0; v < Kv; ++v) {
      const int q = rank_of_vp(v);
      samples[size_t(s) * Kv + v] = all[q * row + size_t(s) * Kv + v];
    }
  }
  keep_walls();
}

void Runtime::step_walls(int64_t first, int32_t n, double* out) const {
  if (n < 0 || first < 0) throw ValidationError("step range out of bounds");
  for (int32_t i = 0; i < n; ++i) {
    const size_t g = size_t(first + i);
    out[i] = g < step_wall_.size() ? step_wall_[g] : std::nan("");
  }
}

void Runtime::require_no_open_window(const char* who) const {
  if (cur_step_ != 0)
    throw RuntimeFault(std::string(who) + ": an epoch started by advance() is still open (" +
                       std::to_string(cur_step_) + " of its steps done); finish it first");
}

void Runtime::step_api(int32_t mode, int32_t epoch_step, double* wall, od_sample* out) {
  if (mode != kSync && mode != kAsync) throw ValidationError("unknown launch mode");
  require_no_open_window("step_time");
  begin_window();
  launch_step(mode, epoch_step, false);
  std::vector<double> walls, samples;
  collect(walls, samples);
  if (wall) *wall = walls[0];
  if (out)
    for (int32_t v = 0; v < K(); ++v) out[v] = od_sample{v, epoch_step, mode, 0, samples[v]};
}

// engine.hpp:235-272 with measured samples and real migration
void Runtime::finish_epoch(int32_t e, int32_t steps, EpochOut& o) {
  const auto tb = std::chrono::steady_clock::now();
  std::vector<double> samples;
  const double tr0 = trace_on() ? now_s() : 0;
  collect(o.walls, samples);
  const double tr1 = trace_on() ? now_s() : 0;
  SampleStore db(K(), cfg_.async_steps, cfg_.sync_steps);
  for (int32_t s = 0; s < steps; ++s) {
    const int32_t mode = s < cfg_.async_steps ? kAsync : kSync;
    for (int32_t v = 0; v < K(); ++v) db.add(v, s, mode, samples[size_t(s) * K() + v]);
  }
  o.loads = db.sync_means();
  Decision d = decide_epoch(o.loads, map_, P(), e, cfg_.epochs, balance_calls_,
                            cfg_.first_call_strategy, cfg_.later_call_strategy,
                            cfg_.trigger_threshold, cfg_.refine_tolerance,
                            cfg_.decomposition_kind, cfg_.kx, cfg_.ky,
                            cfg_.capacity_mib > 0 ? &capacity_ : nullptr);
  o.totals = d.totals;
  o.imb_before = d.imbalance_before;
  o.imb_after = d.imbalance_after;
  o.strategy = d.strategy;
  o.plan = d.plan;
  const double tr2 = trace_on() ? now_s() : 0;
  if (!o.plan.empty()) {
    const auto t0 = std::chrono::steady_clock::now();
    migrate(o.plan);
    o.mig_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  if (trace_on())
    std::fprintf(stderr, "[od rank %d] epoch %d boundary: collect %.3f ms, decide %.3f ms, "
                 "migrate %.3f ms (%zu moves)\n", rank_, e, (tr1 - tr0) * 1e3, (tr2 - tr1) * 1e3,
                 (now_s() - tr2) * 1e3, o.plan.size());
  od_epoch_summary h{};
  h.epoch = e;
  h.strategy = o.strategy;
  h.n_moves = int32_t(o.plan.size());
  h.n_steps = steps;
  for (double w : o.walls) h.compute_total += w;
  h.migration_seconds = o.mig_s;
  h.imbalance_before = o.imb_before;
  h.imbalance_after = o.imb_after;
  h.boundary_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
  history_.push_back(h);
}

void Runtime::run_epoch(int32_t e, od_epoch_record* rec) {
  const int32_t S = cfg_.async_steps + cfg_.sync_steps;
  require_no_open_window("run_epoch");
  EpochOut o;
  o.map_before = map_;
  const double tr0 = trace_on() ? now_s() : 0;
  o.classes = classify();
  begin_window();
  double tr1 = 0;
  for (int32_t s = 0; s < S; ++s) {
    advance_advection(e, s);
    launch_step(s < cfg_.async_steps ? kAsync : kSync, s, false);
    if (s == 0 && trace_on()) {
      tr1 = now_s();
      if (tr_drained_ > 0)
        std::fprintf(stderr, "[od rank %d] epoch %d: GPU idle between epochs (host) %.3f ms\n",
                     rank_, e, (tr1 - tr_drained_) * 1e3);
    }
    ++global_step_;
  }
  if (trace_on())
    std::fprintf(stderr, "[od rank %d] epoch %d start: classify+first launch %.3f ms\n", rank_, e,
                 (tr1 - tr0) * 1e3);
  finish_epoch(e, S, o);
  if (!rec) return;
  rec->epoch = e;
  rec->n_steps = S;
  rec->compute_total = 0;
  for (int32_t s = 0; s < S; ++s) {
    if (rec->step_times) rec->step_times[s] = o.walls[s];
    rec->compute_total += o.walls[s];
  }
  rec->strategy = o.strategy;
  rec->n_moves = int32_t(o.plan.size());
  if (rec->moves) {
    // snprintf convention: n_moves is the plan's size, at most moves_cap moves
    // are written (the epoch, migration included, has been committed either way)
    const size_t m = std::min(o.plan.size(), size_t(std::max(rec->moves_cap, 0)));
    for (size_t i = 0; i < m; ++i)
      rec->moves[i] = od_move{o.plan[i].vp, o.plan[i].from, o.plan[i].to};
  }
  rec->migration_seconds = o.mig_s;
  rec->imbalance_before = o.imb_before;
  rec->imbalance_after = o.imb_after;
  if (rec->proc_loads) std::copy(o.totals.begin(), o.totals.end(), rec->proc_loads);
  if (rec->vp_loads) std::copy(o.loads.begin(), o.loads.end(), rec->vp_loads);
  if (rec->mapping) std::copy(o.map_before.begin(), o.map_before.end(), rec->mapping);
  if (rec->classes) std::copy(o.classes.begin(), o.classes.end(), rec->classes);
}

void Runtime::advance(int32_t n, int32_t* epochs_done) {
  const int32_t S = cfg_.async_steps + cfg_.sync_steps;
  int32_t done = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (cur_step_ == 0) begin_window();
    advance_advection(cur_epoch_, cur_step_);
    launch_step(cur_step_ < cfg_.async_steps ? kAsync : kSync, cur_step_, false);
    ++global_step_;
    if (++cur_step_ == S) {
      EpochOut o;
      finish_epoch(cur_epoch_, S, o);
      ++cur_epoch_;
      cur_step_ = 0;
      ++done;
    }
  }
  if (epochs_done) *epochs_done = done;
}

void Runtime::advance_host(int32_t n, const double* host_c, int32_t n_fields, double* host_loads) {
  if (n < 0) throw ValidationError("negative step count");
  const size_t cells = size_t(cfg_.nx) * cfg_.ny;
  // one mapped slot per window position + 1: a caller's field is staged into
  // slot (global step % (S + 1)) while the previous step runs, so no slot is
  // rewritten while a step kernel that may still be in flight reads it (the
  // host runs at most one epoch ahead: epoch ends drain the stream)
  const int32_t Sw = std::max(cfg_.async_steps + cfg_.sync_steps, 1) + 1;
  if (int32_t(h_ring_.size()) < Sw) {
    OD_CU(cudaStreamSynchronize(s0_));
    while (int32_t(h_ring_.size()) < Sw) {
      double* h = nullptr;
      double* d = nullptr;
      OD_CU(cudaHostAlloc(reinterpret_cast<void**>(&h), cells * sizeof(double), cudaHostAllocMapped));
      OD_CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0));
      h_ring_.push_back(h);
      d_ring_.push_back(d);
    }
  }
  if (!h_cstage_[0]) {
    for (int b = 0; b < 2; ++b) {
      OD_CU(cudaMallocHost(&h_cstage_[b], cells * sizeof(double)));
      OD_CU(cudaMalloc(&d_cstage_[b], cells * sizeof(double)));
      OD_CU(cudaEventCreateWithFlags(&cstage_ev_[b], cudaEventDisableTiming));
    }
  }
  const size_t row_words = 2 * std::max<size_t>(K(), 1);
  if (h_loads_rows_ < size_t(std::max(n, 1))) {
    OD_CU(cudaStreamSynchronize(s0_));
    if (h_loads_) cudaFreeHost(h_loads_);
    h_loads_rows_ = size_t(std::max(n, 1));
    OD_CU(cudaHostAlloc(reinterpret_cast<void**>(&h_loads_),
                        h_loads_rows_ * row_words * sizeof(unsigned long long), cudaHostAllocMapped));
    OD_CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_loads_map_), h_loads_, 0));
  }
  if (n_fields < 0 || (n_fields > 0 && !host_c)) throw ValidationError("bad host field count");
  const int32_t S = cfg_.async_steps + cfg_.sync_steps;
  // steps are launched back to back; the per-step loads land in pinned rows
  // and are read once the stream has drained (epoch ends drain it anyway)
  std::vector<std::vector<int32_t>> step_vps(host_loads ? n : 0);
  const bool caller = host_c && n_fields > 0;
  auto field_of = [&](int32_t i) { return host_c + size_t(std::min(i, n_fields - 1)) * cells; };
  const size_t ring_n = h_ring_.size();
  // staging of caller fields, one step ahead: the copy into the mapped slot and
  // the change test (for the tile order) run while the GPU works on the
  // previous step -- also across epoch ends, where the stream drains
  std::vector<char> changed(caller ? n : 0, 0);
  const size_t base_g = size_t(global_step_);  // step i is global step base_g + i
  auto stage = [&](int32_t i) {
    const double* f = field_of(i);
    std::memcpy(h_ring_[(base_g + size_t(i)) % ring_n], f, cells * sizeof(double));
    if (i == 0)
      changed[i] = std::memcmp(field_.c.data(), f, cells * sizeof(double)) != 0;
    else
      changed[i] = f != field_of(i - 1) &&
                   std::memcmp(field_of(i - 1), f, cells * sizeof(double)) != 0;
  };
  if (caller && n > 0) stage(0);
  for (int32_t i = 0; i < n; ++i) {
    if (cur_step_ == 0) begin_window();
    const uint64_t gen0 = field_gen_;
    advance_advection(cur_epoch_, cur_step_);  // (may reset field_ to the runtime's own)
    const bool reset = field_gen_ != gen0;
    h_loads_dst_ = h_loads_ + size_t(i) * row_words;
    d_loads_dst_ = d_loads_map_ + size_t(i) * row_words;
    const double* hf = nullptr;
    int slot = -1;
    if (caller) {
      // the caller's field for this step drives the kernel; the host-side copy
      // of it orders the tiles (heaviest first) when it differs from the last
      hf = field_of(i);
      slot = int((base_g + size_t(i)) % ring_n);
      if (changed[i] || reset) {
        field_.c.assign(hf, hf + cells);
        ++field_gen_;
        order_dirty_ = true;
      }
    }
    launch_step(cur_step_ < cfg_.async_steps ? kAsync : kSync, cur_step_, true, hf, slot);
    if (caller && i + 1 < n) stage(i + 1);
    if (host_loads) step_vps[i] = window_.back().slot_vps;
    ++global_step_;
    if (++cur_step_ == S) {
      EpochOut o;
      finish_epoch(cur_epoch_, S, o);
      ++cur_epoch_;
      cur_step_ = 0;
    }
  }
  // later steps see the runtime's own advected field again
  if (host_c && n_fields > 0) set_shift(shift_);
  OD_CU(cudaStreamSynchronize(s0_));
  for (int32_t i = 0; host_loads && i < n; ++i) {
    double* row = host_loads + size_t(i) * K();
    std::fill(row, row + K(), 0.0);
    const unsigned long long* src = h_loads_ + size_t(i) * row_words;
    for (size_t j = 0; j < step_vps[i].size(); ++j) row[step_vps[i][j]] = double(src[2 * j]) * 1e-9;
  }
}

// ---------------------------------------------------------------- migrate --

void Runtime::migrate(const std::vector<MoveRec>& plan) {
  const double t0 = now_s();
  std::vector<int32_t> next = apply_moves(map_, P(), plan);  // throws before any data moves
  double t1 = t0, t2 = t0, t3 = t0;
  if (world_ > 1) {
    std::vector<int32_t> moved;
    for (int32_t v = 0; v < K(); ++v)
      if (rank_of_proc(map_[v]) != rank_of_proc(next[v])) moved.push_back(v);
    std::vector<ChunkMem> incoming(K());
    for (int32_t v : moved)
      if (rank_of_proc(next[v]) == rank_) incoming[v] = alloc_chunk(v);
    OD_CU(cudaStreamSynchronize(s0_));
    t1 = now_s();
    // where every chunk lives in its owner's slab (elements; -1: outside the slab)
    bool pulled = false;
    if (p2p_ && peer_slabs_ok_ && !moved.empty() && !std::getenv("OD_MIGRATE_NCCL")) {
      std::vector<int64_t> mine(K(), -1);
      const int64_t slab_elems = int64_t(slab_slots_ * (slot_bytes_ / sizeof(double)));
      for (int32_t v = 0; v < K(); ++v)
        if (rank_of_proc(map_[v]) == rank_ && chunks_[v].base && chunks_[v].base >= slab_ &&
            chunks_[v].base < slab_ + slab_elems)
          mine[v] = int64_t(chunks_[v].base - slab_);
      // migration scratch (offsets, pull jobs, ordering word) allocated once: a
      // cudaMalloc/cudaFree pair per epoch would synchronise the device each time
      if (!d_mig_off_) {
        OD_CU(cudaMalloc(&d_mig_off_, sizeof(int64_t) * size_t(K()) * (world_ + 1)));
        OD_CU(cudaMalloc(&d_mig_jobs_, sizeof(CopyJob) * 2 * size_t(K())));
        OD_CU(cudaMalloc(&d_mig_one_, sizeof(int32_t)));
      }
      int64_t* d_off = d_mig_off_;
      OD_CU(cudaMemcpyAsync(d_off, mine.data(), sizeof(int64_t) * K(), cudaMemcpyHostToDevice,
                            s0_));
      OD_NC(odb::nccl().AllGather(d_off, d_off + K(), size_t(K()), ncclInt64, comm_, s0_));
      std::vector<int64_t> all(size_t(K()) * world_);
      OD_CU(cudaMemcpyAsync(all.data(), d_off + K(), sizeof(int64_t) * all.size(),
                            cudaMemcpyDeviceToHost, s0_));
      OD_CU(cudaStreamSynchronize(s0_));
      bool ok = true;
      for (int32_t v : moved) ok = ok && all[size_t(rank_of_proc(map_[v])) * K() + v] >= 0;
      if (ok) {
        // the new owner pulls U^t and A straight out of the old owner's slab over
        // NVLink (copy engines, all pairs concurrently), then every rank waits
        // for every pull before any source slot is reused
        std::vector<CopyJob> pulls;
        for (int32_t v : moved) {
          const int src = rank_of_proc(map_[v]), dst = rank_of_proc(next[v]);
          const size_t plane = size_t(subs_[v].h()) * ((subs_[v].w() + 15) / 16 * 16);
          const size_t ae = plane * cfg_.nz, fe = ae * cfg_.fields;
          if (src == rank_) st_.migrated_bytes += int64_t((fe + ae) * sizeof(double));
          if (dst != rank_) continue;
          const double* sb = peer_slab_[src] + all[size_t(src) * K() + v];
          const ChunkMem& in = incoming[v];
          pulls.push_back(CopyJob{sb + (in.u[parity_] - in.base), in.u[parity_], int64_t(fe)});
          pulls.push_back(CopyJob{sb + (in.a - in.base), in.a, int64_t(ae)});
        }
        if (!pulls.empty()) {
          CopyJob* d_jobs = d_mig_jobs_;
          OD_CU(cudaMemcpyAsync(d_jobs, pulls.data(), pulls.size() * sizeof(CopyJob),
                                cudaMemcpyHostToDevice, s0_));
          // ~2 waves of 256-thread CTAs spread over the jobs
          const unsigned per_job = std::max(1u, unsigned(2 * 148 * 8 / pulls.size()));
          pull_chunks<<<dim3(per_job, unsigned(pulls.size())), 256, 0, s0_>>>(d_jobs);
          OD_CU(cudaGetLastError());
          ++st_.kernel_launches;
        }
        // (stream order: the all-reduce runs after this rank's pulls)
        int32_t* d_one = d_mig_one_;
        OD_CU(cudaMemsetAsync(d_one, 0, sizeof(int32_t), s0_));
        OD_NC(odb::nccl().AllReduce(d_one, d_one, 1, ncclInt32, ncclSum, comm_, s0_));
        OD_CU(cudaStreamSynchronize(s0_));
        pulled = true;
      }
    }
    if (!pulled) OD_NC(odb::nccl().GroupStart());
    for (int32_t v : moved) {
      if (pulled) break;
      const int src = rank_of_proc(map_[v]), dst = rank_of_proc(next[v]);
      const size_t plane = size_t(subs_[v].h()) * ((subs_[v].w() + 15) / 16 * 16);
      const size_t ae = plane * cfg_.nz, fe = ae * cfg_.fields;
      if (src == rank_) {
        OD_NC(odb::nccl().Send(chunks_[v].u[parity_], fe, ncclFloat64, dst, comm_, s0_));
        OD_NC(odb::nccl().Send(chunks_[v].a, ae, ncclFloat64, dst, comm_, s0_));
        st_.migrated_bytes += int64_t((fe + ae) * sizeof(double));
      }
      if (dst == rank_) {
        OD_NC(odb::nccl().Recv(incoming[v].u[parity_], fe, ncclFloat64, src, comm_, s0_));
        OD_NC(odb::nccl().Recv(incoming[v].a, ae, ncclFloat64, src, comm_, s0_));
      }
    }
    if (!pulled) OD_NC(odb::nccl().GroupEnd());
    OD_CU(cudaStreamSynchronize(s0_));
    t2 = now_s();
    for (int32_t v : moved) {
      if (rank_of_proc(map_[v]) == rank_) release_chunk(chunks_[v]);
      if (rank_of_proc(next[v]) == rank_) chunks_[v] = incoming[v];
    }
  }
  map_ = std::move(next);
  t3 = now_s();
  rebuild_tables();
  if (trace_on())
    fprintf(stderr, "[od rank %d] migrate: alloc+sync %.2f ms, transfer %.2f ms, release %.2f ms, "
            "rebuild %.2f ms, moves %zu\n", rank_, (t1 - t0) * 1e3, (t2 - t1) * 1e3,
            (t3 - t2) * 1e3, (now_s() - t3) * 1e3, plan.size());
}

bool Runtime::read_chunk(int32_t vp, double* u, double* a) {
  if (vp < 0 || vp >= K()) throw ValidationError("vp out of range");
  if (rank_of_vp(vp) != rank_) return false;
  OD_CU(cudaStreamSynchronize(s0_));
  const ChunkMem& m = chunks_[vp];
  const size_t w = m.sub.w(), h = m.sub.h();
  const size_t rows_u = h * cfg_.nz * cfg_.fields, rows_a = h * cfg_.nz;
  if (u)
    OD_CU(cudaMemcpy2D(u, w * sizeof(double), m.u[parity_], m.pitch * sizeof(double),
                       w * sizeof(double), rows_u, cudaMemcpyDeviceToHost));
  if (a)
    OD_CU(cudaMemcpy2D(a, w * sizeof(double), m.a, m.pitch * sizeof(double), w * sizeof(double),
                       rows_a, cudaMemcpyDeviceToHost));
  return true;
}

void Runtime::stats(od_rt_stats* s) {
  // trips of the current load field over the resident columns (host count)
  int64_t trips = 0;
  for (int32_t v : resident_) {
    const Sub& sb = subs_[v];
    for (int32_t y = sb.y0; y < sb.y1; ++y)
      for (int32_t x = sb.x0; x < sb.x1; ++x) {
        const int32_t t = int32_t(std::floor(double(cfg_.nz) * field_.at(x, y))) - 1;
        trips += t > 0 ? t : 0;
      }
  }
  st_.physics_trips = trips;
  st_.last_kernel = last_kernel_;
  *s = st_;
}

}  // namespace odb

// ----------------------------------------------------------------- C ABI --

using odb::guarded;
using odb::Runtime;
using odb::ValidationError;
using odb::RuntimeFault;

struct od_runtime {
  Runtime* rt;
};

static Runtime& R(const od_runtime* h) {
  if (!h || !h->rt) throw ValidationError("null runtime handle");
  return *h->rt;
}

extern "C" {

int od_nccl_unique_id(uint8_t* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null pointer: out");
    ncclUniqueId id;
    OD_NC(odb::nccl().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
  });
}

int od_rt_create(const od_config* cfg, int32_t rank, int32_t world, int32_t device,
                 const uint8_t* nccl_id, od_runtime** out) {
  return guarded([&] {
    if (!cfg || !out) throw ValidationError("null pointer: cfg/out");
    *out = nullptr;
    auto* h = new od_runtime{nullptr};
    try {
      h->rt = new Runtime(*cfg, rank, world, device, nccl_id);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void od_rt_destroy(od_runtime* rt) {
  if (!rt) return;
  delete rt->rt;
  delete rt;
}

int od_rt_vp_count(const od_runtime* rt, int32_t* k) {
  return guarded([&] { *k = R(rt).K(); });
}

int od_rt_proc_count(const od_runtime* rt, int32_t* p) {
  return guarded([&] { *p = R(rt).P(); });
}

int od_rt_mapping(const od_runtime* rt, int32_t* map) {
  return guarded([&] {
    const auto& m = R(rt).mapping();
    std::copy(m.begin(), m.end(), map);
  });
}

int od_rt_subdomains(const od_runtime* rt, od_subdomain* out) {
  return guarded([&] {
    const auto& s = R(rt).subs();
    for (size_t i = 0; i < s.size(); ++i)
      out[i] = od_subdomain{s[i].vp, s[i].x0, s[i].x1, s[i].y0, s[i].y1, s[i].boundary};
  });
}

int od_rt_classify(const od_runtime* rt, int32_t* classes) {
  return guarded([&] {
    auto c = R(rt).classify();
    std::copy(c.begin(), c.end(), classes);
  });
}

int od_rt_load_field(const od_runtime* rt, double* c) {
  return guarded([&] {
    const auto& f = R(rt).field();
    std::copy(f.c.begin(), f.c.end(), c);
  });
}

int od_rt_step(od_runtime* rt, int32_t mode, int32_t epoch_step, int32_t /*global_step*/,
               double* wall, od_sample* samples) {
  return guarded([&] { R(rt).step_api(mode, epoch_step, wall, samples); });
}

int od_rt_run_epoch(od_runtime* rt, int32_t epoch_index, od_epoch_record* rec) {
  return guarded([&] { R(rt).run_epoch(epoch_index, rec); });
}

int od_rt_advance(od_runtime* rt, int32_t n_steps, int32_t* epochs_done) {
  return guarded([&] { R(rt).advance(n_steps, epochs_done); });
}

int od_rt_advance_host(od_runtime* rt, int32_t n_steps, const double* host_c_fields,
                       int32_t n_fields, double* host_step_loads) {
  return guarded([&] { R(rt).advance_host(n_steps, host_c_fields, n_fields, host_step_loads); });
}

int od_rt_migrate(od_runtime* rt, const od_move* moves, int32_t n_moves) {
  return guarded([&] {
    if (n_moves < 0) throw ValidationError("negative move count");
    std::vector<odb::MoveRec> plan(n_moves);
    for (int32_t i = 0; i < n_moves; ++i) plan[i] = {moves[i].vp, moves[i].from, moves[i].to};
    R(rt).migrate(plan);
  });
}

int od_rt_read_chunk(od_runtime* rt, int32_t vp, double* u, double* a, int32_t* resident) {
  return guarded([&] {
    const bool r = R(rt).read_chunk(vp, u, a);
    if (resident) *resident = r ? 1 : 0;
  });
}

int od_rt_stats_get(od_runtime* rt, od_rt_stats* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null pointer: out");
    R(rt).stats(out);
  });
}

int od_rt_epoch_history(od_runtime* rt, od_epoch_summary* out, int32_t cap, int32_t* n) {
  return guarded([&] {
    const auto& h = R(rt).history();
    if (!n) throw ValidationError("null pointer: n");
    *n = int32_t(h.size());
    const int32_t m = std::min<int32_t>(cap, int32_t(h.size()));
    for (int32_t i = 0; i < m; ++i) out[i] = h[h.size() - m + i];
  });
}

int od_rt_set_profiling(od_runtime* rt, int32_t on) {
  return guarded([&] { R(rt).set_profiling(on != 0); });
}

int od_rt_synchronize(od_runtime* rt) {
  return guarded([&] { R(rt).sync(); });
}

int od_rt_step_walls(od_runtime* rt, int64_t first, int32_t n, double* out) {
  return guarded([&] {
    if (n > 0 && !out) throw ValidationError("null pointer: out");
    R(rt).step_walls(first, n, out);
  });
}

}  // extern "C"
