// Host-side model of the over-decomposed BRAMS-like workload: decomposition,
// load field, chunk->processor mapping, measurement store and the two load
// balancers.  Pure functions on plain vectors, callable from the C ABI
// (od_capi.cpp) and from the device runtime (od_runtime.cu).
//
// Arithmetic that feeds a balancing decision follows the reference's
// operation order exactly so plans are bit-identical for the same loads
// (/root/reference/proj/include/overdeck/{workload,cluster,measurement,
// balancer}.hpp; the file:line of each counterpart is cited per function).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace odb {

// Input-contract violation -> OD_EVALIDATION (errors.hpp:9-12).
struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
// Mid-run failure (stale plan, incomplete measurement, device error)
// -> OD_ERUNTIME (errors.hpp:15-18).
struct RuntimeFault : std::runtime_error {
  explicit RuntimeFault(const std::string& m) : std::runtime_error(m) {}
};

enum Mode : int32_t { kSync = 0, kAsync = 1 };
enum Strategy : int32_t { kGreedy = 0, kRefineSwap = 1, kRefineAdjacent = 2 };
enum VpClass : int32_t { kHeavy = 0, kLight = 1 };
enum Pattern : int32_t { kUniform = 0, kStaticNode0 = 1, kUpperHalfHeavy = 2 };

struct Sub {  // one chunk of columns, half-open ranges
  int32_t vp = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
  int64_t boundary = 0;  // cells on faces shared with another chunk
  int64_t cells() const { return int64_t(x1 - x0) * (y1 - y0); }
  int32_t w() const { return x1 - x0; }
  int32_t h() const { return y1 - y0; }
};

struct MoveRec {
  int32_t vp, from, to;
  bool operator==(const MoveRec& o) const { return vp == o.vp && from == o.from && to == o.to; }
};

struct Work {
  double items = 0, depth = 0;
  double total() const { return items * depth; }
};

// ---- workload ---------------------------------------------------------------
// contiguous pieces, the first extent%k pieces one longer (workload.hpp:85-95)
std::vector<std::pair<int32_t, int32_t>> split_extent(int32_t extent, int32_t pieces);
std::vector<Sub> strips_1d(int32_t nx, int32_t ny, int32_t k);                 // :100-114
std::vector<Sub> tiles_2d(int32_t nx, int32_t ny, int32_t kx, int32_t ky);     // :117-139
void check_domain(int32_t nx, int32_t ny, int32_t nz, int32_t fields);         // :20-23

// Column multiplier C, y-major c[y*nx+x] (workload.hpp:41-71).
struct Field2D {
  int32_t nx = 0, ny = 0;
  std::vector<double> c;
  double at(int32_t x, int32_t y) const { return c[size_t(y) * nx + x]; }
  double mean_over(const Sub& s) const;  // :58-64
};
Field2D make_load_field(int32_t nx, int32_t ny, Pattern p, double heavy, double light,
                        const std::vector<Sub>& node0_subs);          // :160-181
Field2D shift_rows_down(const Field2D& c, int32_t shift);              // :185-195
Work physics_trips(const Sub& s, const Field2D& c, int32_t mzp);       // :199-204
Work jacobi_items(const Sub& s, int32_t nz, int32_t fields);           // :207-210
int64_t halo_footprint(const Sub& s, int32_t nz, int32_t fields);      // :213-215
int64_t chunk_footprint(const Sub& s, int32_t nz, int32_t fields);     // :218-220

// ---- cluster ----------------------------------------------------------------
std::vector<int32_t> block_mapping(int32_t K, int32_t P);              // cluster.hpp:115-127
// all-or-nothing; throws RuntimeFault on the first stale move (:130-139)
std::vector<int32_t> apply_moves(const std::vector<int32_t>& map, int32_t P,
                                 const std::vector<MoveRec>& moves);
std::vector<double> totals_per_proc(const std::vector<double>& loads,
                                    const std::vector<int32_t>& map, int32_t P);  // :142-148
double max_over_mean(const std::vector<double>& totals);              // :151-157

// ---- balancer ---------------------------------------------------------------
bool balance_needed(const std::vector<double>& totals, double threshold);  // balancer.hpp:29-32
std::vector<MoveRec> plan_greedy(const std::vector<double>& loads,
                                 const std::vector<int32_t>& map, int32_t P);  // :36-63
std::vector<MoveRec> plan_refine_swap(const std::vector<double>& loads,
                                      const std::vector<int32_t>& map, int32_t P,
                                      double tol);
// B200 extension (off-parity): refine_swap_lb's rounds and acceptance tests,
// choosing among admissible actions the one adding the fewest cross-processor
// chunk faces (balance score breaks ties); Strategy 2
std::vector<MoveRec> plan_refine_adjacent(const std::vector<double>& loads,
                                          const std::vector<int32_t>& map, int32_t P, double tol,
                                          int32_t kind, int32_t kx, int32_t ky);                            // :68-152

// B200 extension (off-parity): capacity-aware balancing.  The reference's
// balancers ignore memory: GreedyLB can pack chunks onto one GPU
// past its HBM.  Processors are grouped into bins (the GPUs that hold them);
// a plan never moves a chunk into a bin whose resident chunk bytes would then
// exceed its capacity (moves out of an over-full bin are always allowed).
// With capacities no plan can reach, both equal plan_greedy /
// plan_refine_swap exactly.
struct Capacity {
  std::vector<int64_t> vp_bytes;     // K
  std::vector<int32_t> bin_of_proc;  // P
  std::vector<int64_t> bin_cap;      // bins
  void validate(int32_t K, int32_t P) const;
};
std::vector<MoveRec> plan_greedy_capacity(const std::vector<double>& loads,
                                          const std::vector<int32_t>& map, int32_t P,
                                          const Capacity& cap);
std::vector<MoveRec> plan_refine_capacity(const std::vector<double>& loads,
                                          const std::vector<int32_t>& map, int32_t P, double tol,
                                          const Capacity& cap);

// ---- modelled costs (gpu_cost.hpp:21-80, balancer.hpp:157-175) ---------------
// The B200 path measures these quantities; the model functions stay available
// with the reference's arithmetic for users who compare against the simulator.
struct GpuCostModel {
  double launch_overhead = 1.0e-4, per_item_time = 1.0e-9, saturation_floor = 0.0;
  double h2d_bandwidth = 6.0e9, d2h_bandwidth = 6.0e9, async_overlap_gain = 0.06;
  void validate() const;
};
double kernel_time_sync_model(const Work& w, const GpuCostModel& g);                // :50-54
double transfer_time_model(double bytes, bool host_to_device, const GpuCostModel& g);  // :60-66
double node_gpu_schedule_model(const std::vector<double>& jobs, int32_t mode,
                               const GpuCostModel& g);                                // :70-80
// plan_cost: per moved VP a D2H stage on the source node, an H2D stage on the
// destination node, plus the network hop on both when the nodes differ; nodes
// in parallel, each node's transfers serialised (balancer.hpp:157-175)
double plan_cost_model(const std::vector<MoveRec>& plan, const std::vector<int64_t>& data_bytes,
                       int32_t procs_per_node, int32_t nodes, double net_bandwidth,
                       double net_latency, const GpuCostModel& g);

// B200 migration cost (replaces plan_cost's host staging, balancer.hpp:157-175):
// a chunk moves as one peer copy between the two GPUs owning its old and new
// processor (procs_per_gpu processors per GPU; moves inside a GPU are free).
// GPUs copy concurrently; a GPU's sends and receives share its NVLink port, so
// the plan costs max over GPUs of max(bytes out, bytes in) / link_bandwidth
// plus latency per transfer touching that GPU.
double plan_cost_nvlink_model(const std::vector<MoveRec>& plan,
                              const std::vector<int64_t>& data_bytes, int32_t procs_per_gpu,
                              int32_t gpus, double link_bandwidth, double latency);

// ---- calibration (gpu_cost.hpp:82-258, engine.hpp:363-373) -----------------
struct CalibSample {
  Work w;
  double seconds = 0;
};
struct GpuFit {
  GpuCostModel model;
  double max_rel_residual = 0;
};
// calibrate_gpu: rows within 10 % of the fastest are the saturated floor, the
// others get a least-squares line; if that leaves a residual, a Nelder-Mead
// pass on (launch, rate, floor) minimises the squared relative error of the
// full hinge model and is kept when it is better
GpuFit calibrate_gpu_model(const std::vector<CalibSample>& samples, const GpuCostModel& defaults);
// calibrate_cpu: least squares through the origin (per-item seconds)
double calibrate_cpu_model(const std::vector<CalibSample>& samples);
double cpu_time_model(const Work& w, double cpu_per_item);
// scaling_probe: an n x m grid with an `inner`-deep serial loop per interior
// point, for each m: (cpu seconds, gpu seconds) under the two models
void scaling_probe_model(int32_t n, const std::vector<int32_t>& m_list, double inner,
                         const GpuCostModel& g, double cpu_per_item, std::vector<double>& cpu_s,
                         std::vector<double>& gpu_s);

// ---- epoch policy (Engine::run_epoch, engine.hpp:257-268) --------------------
struct Decision {
  int32_t strategy = -1;  // -1: no strategy called
  std::vector<MoveRec> plan;
  std::vector<double> totals;
  double imbalance_before = 1, imbalance_after = 1;
};
// Given the epoch's per-VP loads: totals, imbalance, trigger check (never on
// the last epoch), first call -> first strategy, later calls -> later
// strategy; balance_calls is incremented on every triggered call.
// With `cap`, Greedy and RefineSwap calls use the capacity-aware planners.
Decision decide_epoch(const std::vector<double>& loads, const std::vector<int32_t>& map,
                      int32_t P, int32_t epoch, int32_t epochs, int32_t& balance_calls,
                      int32_t first_strategy, int32_t later_strategy, double threshold,
                      double tolerance, int32_t kind = -1, int32_t kx = 0, int32_t ky = 0,
                      const Capacity* cap = nullptr);

// ---- halo exchange schedule -------------------------------------------------
// Faces between chunks owned by different ranks.  Both sides enumerate the
// faces in (sender vp, side) order, so the packed buffers line up without any
// metadata exchange.  Layout of one face: [field][level][position], row
// stride lenp = len rounded up to even (16-byte aligned pairs).
struct FaceXfer {
  int32_t peer, vp, side, nbr, len, lenp;  // vp: owner of the strip (sender side)
  int64_t offset;                          // element offset in the send/recv buffer
};
// Neighbour of vp across `side` (0 left, 1 right, 2 top, 3 bottom) or -1.
int32_t chunk_neighbor(int32_t kind, int32_t kx, int32_t ky, int32_t vp, int32_t side);
void exchange_schedule(const std::vector<Sub>& subs, int32_t kind, int32_t kx, int32_t ky,
                       const std::vector<int32_t>& rank_of_vp, int32_t world, int32_t rank,
                       int64_t per_cell, std::vector<FaceXfer>& sends,
                       std::vector<FaceXfer>& recvs);

// ---- measurement --------------------------------------------------------------
// Per-epoch sample store (measurement.hpp:40-70) + epoch_loads (:75-91).
class SampleStore {
 public:
  SampleStore(int32_t K, int32_t async_steps, int32_t sync_steps);
  void add(int32_t vp, int32_t step, int32_t mode, double value);
  void reset();
  std::vector<double> sync_means() const;
  int32_t vp_count() const { return K_; }
  size_t size() const { return rec_.size(); }

 private:
  struct Rec { int32_t vp, step, mode; double v; };
  int32_t K_, async_, sync_;
  std::vector<Rec> rec_;
  std::vector<uint8_t> seen_;  // K x epoch_steps occupancy
};

// splitmix64 finaliser (public-domain mixer; engine.hpp:112-118 uses it too)
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace odb
