/*
 * overdeck_b200.h -- C ABI of the B200-native BRAMS-like column-update path
 * with Charm++/AMPI-style over-decomposition and dynamic load balancing.
 *
 * Every entry point here replaces one symbol of the reference simulator
 * `overdeck` (headers under /root/reference/proj/include/overdeck/).  The reference is
 * a header-only C++20 library whose API is free functions and value types;
 * the cited file:line is the symbol a binding for this path would call.
 *
 * Conventions
 *  - Plain pointers and sizes only; the caller owns every buffer.
 *  - Return code: OD_OK (0), OD_EVALIDATION (2) for the reference's
 *    ValidationError, OD_ERUNTIME (3) for RuntimeFault and any CUDA/NCCL
 *    failure.  These are the CLI exit codes of tools/main.cpp:17-19.
 *    Nothing throws across this boundary; od_last_error() returns the
 *    message of the last failing call on the calling thread.
 *  - Enumerations keep the reference's declaration order:
 *      LaunchMode  Sync=0 Async=1            (gpu_cost.hpp:15)
 *      Strategy    Greedy=0 RefineSwap=1     (cluster.hpp:69)
 *      VpClass     Heavy=0 Light=1           (cluster.hpp:47)
 *      LoadPattern Uniform=0 StaticNode0=1 UpperHalfHeavy=2 (workload.hpp:141)
 *      DecompositionKind OneD=0 TwoD=1       (engine.hpp:18)
 *  - The pure functions (workload, cluster, measurement, balancer) are
 *    reentrant.  An od_runtime handle is driven by one host thread.
 */
#ifndef OVERDECK_B200_H
#define OVERDECK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OD_OK = 0, OD_EVALIDATION = 2, OD_ERUNTIME = 3 };
enum { OD_SYNC = 0, OD_ASYNC = 1 };
enum { OD_GREEDY = 0, OD_REFINE_SWAP = 1, OD_REFINE_ADJACENT = 2 /* B200 extension */ };
enum { OD_HEAVY = 0, OD_LIGHT = 1 };
enum { OD_UNIFORM = 0, OD_STATIC_NODE0 = 1, OD_UPPER_HALF_HEAVY = 2 };
enum { OD_ONE_D = 0, OD_TWO_D = 1 };
/* per-chunk load measurement in Sync steps */
enum {
  OD_MEASURE_EVENTS = 0,   /* paper protocol: one launch per chunk, cudaEvent pair */
  OD_MEASURE_TIMER = 1,    /* batched launch; per-chunk processor-sharing SM time (in-kernel
                              per-SM clock) apportions the GPU's event-timed kernel time
                              (per-GPU sums = busy time) */
  OD_MEASURE_TIMER_RAW = 2, /* batched launch, raw per-chunk SM-time shares */
  OD_MEASURE_OPS = 3       /* batched launch; in-kernel counted FP64 instructions per chunk
                              apportion the GPU's kernel time (ignores HBM time) */
};

/* Move{vp, from, to}                                   cluster.hpp:62-67 */
typedef struct od_move {
  int32_t vp, from, to;
} od_move;

/* SubDomain: half-open column ranges, shared-face count workload.hpp:29-38 */
typedef struct od_subdomain {
  int32_t owner_vp, x_begin, x_end, y_begin, y_end;
  int64_t boundary_cells;
} od_subdomain;

/* StepSample{vp, step (0-based in epoch), mode, seconds} measurement.hpp:14-19 */
typedef struct od_sample {
  int32_t vp, step, mode, pad_;
  double value;
} od_sample;

/* KernelWork{work_items, serial_depth}                   workload.hpp:75-80 */
typedef struct od_kernel_work {
  double work_items, serial_depth;
} od_kernel_work;

const char* od_last_error(void);
int32_t od_abi_version(void);

/* ---------------------------------------------------------------- workload */
/* decompose_1d                                        workload.hpp:100-114 */
int od_decompose_1d(int32_t nx, int32_t ny, int32_t k, od_subdomain* out /* k */);
/* decompose_2d                                        workload.hpp:117-139 */
int od_decompose_2d(int32_t nx, int32_t ny, int32_t kx, int32_t ky,
                    od_subdomain* out /* kx*ky */);
/* init_load_field; out is y-major c[y*nx+x]           workload.hpp:160-181 */
int od_init_load_field(int32_t nx, int32_t ny, int32_t pattern, double heavy_value,
                       double light_value, const od_subdomain* node0_subs,
                       int32_t n_node0, double* out /* nx*ny */);
/* advect_load_field                                   workload.hpp:185-195 */
int od_advect_load_field(const double* c, int32_t nx, int32_t ny, int32_t shift_rows,
                         double* out /* nx*ny */);
/* LoadField::mean_over                                  workload.hpp:58-64 */
int od_mean_over(const double* c, int32_t nx, int32_t ny, const od_subdomain* sub,
                 double* out);
/* physics_work                                        workload.hpp:199-204 */
int od_physics_work(const od_subdomain* sub, const double* c, int32_t nx, int32_t ny,
                    int32_t mzp, od_kernel_work* out);
/* jacobi_work                                         workload.hpp:207-210 */
int od_jacobi_work(const od_subdomain* sub, int32_t nz, int32_t fields,
                   od_kernel_work* out);
/* halo_bytes / subdomain_bytes (8-byte values)        workload.hpp:213-220 */
int od_halo_bytes(const od_subdomain* sub, int32_t nz, int32_t fields, int64_t* out);
int od_subdomain_bytes(const od_subdomain* sub, int32_t nz, int32_t fields, int64_t* out);

/* ----------------------------------------------------------------- cluster */
/* initial_block_mapping                               cluster.hpp:115-127 */
int od_initial_block_mapping(int32_t vp_count, int32_t proc_count, int32_t* map /* K */);
/* apply_plan: all-or-nothing; map_out untouched on error cluster.hpp:130-139 */
int od_apply_plan(const int32_t* map_in, int32_t vp_count, int32_t proc_count,
                  const od_move* moves, int32_t n_moves, int32_t* map_out /* K */);
/* proc_loads                                          cluster.hpp:142-148 */
int od_proc_loads(const double* loads, int32_t n_loads, const int32_t* map,
                  int32_t vp_count, int32_t proc_count, double* totals /* P */);
/* imbalance_ratio                                     cluster.hpp:151-157 */
int od_imbalance_ratio(const double* totals, int32_t n, double* out);

/* ---------------------------------------------------------- modelled costs */
/* The reference's analytic GPU model (gpu_cost.hpp:21-47).  The B200 path
 * measures instead; these keep the simulator's arithmetic for comparisons. */
typedef struct od_gpu_model {
  double launch_overhead, per_item_time, saturation_floor;
  double h2d_bandwidth, d2h_bandwidth, async_overlap_gain;
} od_gpu_model;
/* kernel_time_sync                                     gpu_cost.hpp:50-54 */
int od_kernel_time_sync(const od_kernel_work* work, const od_gpu_model* gpu, double* out);
/* transfer_time (host_to_device: 1 = H2D, 0 = D2H)      gpu_cost.hpp:60-66 */
int od_transfer_time(double bytes, int32_t host_to_device, const od_gpu_model* gpu, double* out);
/* node_gpu_schedule (mode OD_SYNC / OD_ASYNC)           gpu_cost.hpp:70-80 */
int od_node_gpu_schedule(const double* jobs, int32_t n, int32_t mode, const od_gpu_model* gpu,
                         double* out);
/* plan_cost over per-VP data bytes                     balancer.hpp:157-175 */
int od_plan_cost(const od_move* moves, int32_t n_moves, const int64_t* data_bytes,
                 int32_t vp_count, int32_t procs_per_node, int32_t nodes,
                 double network_bandwidth, double network_latency, const od_gpu_model* gpu,
                 double* out);

/* B200 replacement of plan_cost (balancer.hpp:157-175; no host staging): chunk
   moves are NVLink peer copies between the owning GPUs, GPUs copy concurrently,
   a GPU's sends and receives share its port: max over GPUs of max(bytes out,
   bytes in) / link_bandwidth + latency per transfer touching it.  Moves between
   processors of one GPU are free. */
int od_plan_cost_nvlink(const od_move* moves, int32_t n_moves, const int64_t* data_bytes,
                        int32_t vp_count, int32_t procs_per_gpu, int32_t gpus,
                        double link_bandwidth, double latency, double* out);
/* calibrate_gpu: saturated rows (within 10 % of the fastest) set the floor, a
   least-squares line the rest, then a Nelder-Mead refinement of the hinge model
   when it leaves a residual; non-model fields come from `defaults`
                                                        gpu_cost.hpp:187-246 */
int od_calibrate_gpu(const od_kernel_work* work, const double* seconds, int32_t n,
                     const od_gpu_model* defaults, od_gpu_model* out, double* max_rel_residual);
/* calibrate_cpu: least squares through the origin      gpu_cost.hpp:249-261 */
int od_calibrate_cpu(const od_kernel_work* work, const double* seconds, int32_t n,
                     double* per_item_time);
/* cpu_time                                             gpu_cost.hpp:56-58 */
int od_cpu_time(const od_kernel_work* work, double per_item_time, double* out);
/* scaling_probe: (n-2)*(m-2) items x `inner` per m     engine.hpp:363-373 */
int od_scaling_probe(int32_t n, const int32_t* m_list, int32_t n_m, double inner,
                     const od_gpu_model* gpu, double cpu_per_item, double* cpu_seconds,
                     double* gpu_seconds);

/* ---------------------------------------------------------------- balancer */
/* should_balance                                       balancer.hpp:29-32 */
int od_should_balance(const double* totals, int32_t n, double trigger_threshold,
                      int32_t* out);
/* greedy_lb; moves in ascending vp order; cap >= K     balancer.hpp:36-63 */
int od_greedy_lb(const double* loads, int32_t n_loads, const int32_t* map,
                 int32_t vp_count, int32_t proc_count, od_move* out, int32_t cap,
                 int32_t* n_out);
/* refine_swap_lb; a swap is two moves; cap >= 2*K*P   balancer.hpp:68-152 */
int od_refine_swap_lb(const double* loads, int32_t n_loads, const int32_t* map,
                      int32_t vp_count, int32_t proc_count, double tolerance,
                      od_move* out, int32_t cap, int32_t* n_out);
/* B200 extension, off-parity (no reference counterpart): capacity-aware
   greedy_lb / refine_swap_lb (balancer.hpp:36-152 ignore memory).
   Processors are grouped into bins (the GPUs holding them, bin_of_proc[P]);
   no plan takes a bin's resident chunk bytes (vp_bytes[K]) past
   bin_capacity[n_bins] when the bins fit before it (moves out of an
   over-full bin stay allowed).  Same order, ties and acceptance tests as the
   plain planners, which they equal exactly when no capacity binds; greedy
   places each chunk on the least-loaded processor with room, and if its pass
   still overfills a bin, chunks that moved in return home, lightest first.
   cap >= K (greedy) / 2*K*P (refine). */
int od_greedy_lb_capacity(const double* loads, int32_t n_loads, const int32_t* map,
                          int32_t vp_count, int32_t proc_count, const int64_t* vp_bytes,
                          const int32_t* bin_of_proc, int32_t n_bins,
                          const int64_t* bin_capacity, od_move* out, int32_t cap,
                          int32_t* n_out);
int od_refine_swap_lb_capacity(const double* loads, int32_t n_loads, const int32_t* map,
                               int32_t vp_count, int32_t proc_count, double tolerance,
                               const int64_t* vp_bytes, const int32_t* bin_of_proc,
                               int32_t n_bins, const int64_t* bin_capacity, od_move* out,
                               int32_t cap, int32_t* n_out);
/* B200 extension, off-parity (no reference counterpart; Strategy 2): refine_swap_lb's
   rounds, thresholds and acceptance tests, choosing among admissible moves/swaps the
   one adding the fewest chunk faces between processors (balance score breaks ties);
   decomposition as in od_config; cap >= 2*K*P */
int od_refine_adjacent_lb(const double* loads, int32_t n_loads, const int32_t* map,
                          int32_t vp_count, int32_t proc_count, double tolerance,
                          int32_t decomposition_kind, int32_t kx, int32_t ky, od_move* out,
                          int32_t cap, int32_t* n_out);

/* Engine::run_epoch decision (engine.hpp:257-268) on given per-VP loads:
 * totals, imbalance before/after, trigger (never on the last epoch), first
 * triggered call -> first strategy, later -> later strategy.  *balance_calls
 * is read and incremented on every triggered call.  *strategy = -1 when no
 * strategy was called. */
int od_epoch_decision(const double* loads, int32_t n_loads, const int32_t* map,
                      int32_t vp_count, int32_t proc_count, int32_t epoch_index,
                      int32_t epochs, int32_t* balance_calls, int32_t first_strategy,
                      int32_t later_strategy, double trigger_threshold,
                      double refine_tolerance, int32_t* strategy, od_move* moves,
                      int32_t cap, int32_t* n_moves, double* totals /* P */,
                      double* imbalance_before, double* imbalance_after);

/* ------------------------------------------------------------ halo exchange */
/* Face of a chunk bordering a chunk on another rank (B200 path; the reference
 * models this traffic at engine.hpp:207-217).  Layout of a packed strip:
 * [field][level][position], row stride lenp (len rounded up to even). */
typedef struct od_face_xfer {
  int32_t peer, vp, side, nbr, len, lenp;  /* vp owns the strip; side 0 L 1 R 2 T 3 B */
  int64_t offset;                          /* elements into the send / recv buffer */
} od_face_xfer;
/* neighbour of vp across side, -1 at the domain edge   engine.hpp:290-309 */
int od_chunk_neighbor(int32_t kind, int32_t kx, int32_t ky, int32_t vp, int32_t side,
                      int32_t* out);
int od_exchange_schedule(const od_subdomain* subs, int32_t vp_count, int32_t kind,
                         int32_t kx, int32_t ky, const int32_t* rank_of_vp, int32_t world,
                         int32_t rank, int64_t per_cell, od_face_xfer* sends, int32_t send_cap,
                         int32_t* n_sends, od_face_xfer* recvs, int32_t recv_cap,
                         int32_t* n_recvs);

/* ------------------------------------------------------------- measurement */
/* LoadDB                                             measurement.hpp:40-70 */
typedef struct od_loaddb od_loaddb;
int od_loaddb_create(int32_t vp_count, int32_t async_steps, int32_t sync_steps,
                     od_loaddb** out);
int od_loaddb_record(od_loaddb* db, const od_sample* sample);
int od_loaddb_clear(od_loaddb* db);
int od_loaddb_size(const od_loaddb* db, int32_t* n);
/* epoch_loads: mean of Sync samples only             measurement.hpp:75-91 */
int od_loaddb_epoch_loads(const od_loaddb* db, double* out /* K */);
void od_loaddb_destroy(od_loaddb* db);

/* ----------------------------------------------------------------- runtime */
/*
 * ExperimentConfig (engine.hpp:43-83) restricted to what the B200 path uses.
 * Cluster mapping: one node per GPU (one rank per GPU, world == nodes);
 * procs_per_node processors share a node's GPU exactly as the reference's
 * ClusterSpec (cluster.hpp:18-32).  GpuModel/CpuModel are not present: the
 * B200 path measures instead of modelling.
 */
typedef struct od_config {
  int32_t nodes, procs_per_node;
  int32_t nx, ny, nz, fields;
  int32_t decomposition_kind, kx, ky;
  int32_t async_steps, sync_steps;
  int32_t epochs;
  int32_t pattern;
  double heavy_value, light_value;
  int32_t adv_total_shift_rows, adv_epoch, adv_duration_steps;
  int32_t first_call_strategy, later_call_strategy;
  double trigger_threshold, refine_tolerance;
  uint64_t seed;
  /* B200 path parameters (no reference counterpart) */
  int32_t n_inner;      /* FMA micro-steps per physics trip (f cost), >= 0 */
  int32_t measure;      /* OD_MEASURE_EVENTS | _TIMER | _TIMER_RAW | _OPS */
  int32_t overlap;      /* kernel mode: 0 separate jacobi_step + physics_step;
                           4 fused interleaved tiles (column_step_grid); 5 (default)
                           and 7 warp-specialised tiles (column_step_ws; 5 kept as
                           the default's name from round 1, when it switched between
                           the two by tile count).  Fused modes overlap consecutive
                           step kernels (programmatic dependent launch) */
  int32_t capacity_mib;  /* per-GPU cap on resident chunk data (MiB, B200 extension):
                            > 0 makes the epoch's Greedy / RefineSwap calls
                            capacity-aware (od_*_lb_capacity, one bin per GPU);
                            0 = unlimited, the reference's behaviour */
  int32_t reserved_[4];
} od_config;

/* EpochRecord (engine.hpp:85-97); arrays are caller-allocated */
typedef struct od_epoch_record {
  int32_t epoch;
  int32_t n_steps;           /* out */
  double* step_times;        /* in: cap >= epoch_steps; seconds, max over ranks */
  double compute_total;      /* out: sum of step_times */
  int32_t strategy;          /* out: OD_GREEDY / OD_REFINE_SWAP, -1 = no call */
  int32_t n_moves;           /* out */
  od_move* moves;            /* in: cap moves_cap; min(n_moves, moves_cap) are written */
  int32_t moves_cap;         /* n_moves > moves_cap signals a truncated copy (snprintf
                                convention); the epoch and its migration are committed */
  double migration_seconds;  /* out: measured device time of the chunk moves */
  double imbalance_before, imbalance_after;
  double* proc_loads;        /* in: P */
  double* vp_loads;          /* in: K */
  int32_t* mapping;          /* in: K, mapping active during the epoch */
  int32_t* classes;          /* in: K */
} od_epoch_record;

typedef struct od_runtime od_runtime;

/* NCCL unique id for multi-rank runtimes (rank 0 creates, caller broadcasts) */
int od_nccl_unique_id(uint8_t* out /* 128 bytes */);
/*
 * Engine ctor (engine.hpp:135-157) on the local GPU `device`: decomposition,
 * block mapping, load field, chunk allocation and seeded initial fields.
 * world > 1 needs the NCCL id from od_nccl_unique_id on every rank.
 */
int od_rt_create(const od_config* cfg, int32_t rank, int32_t world, int32_t device,
                 const uint8_t* nccl_id, od_runtime** out);
void od_rt_destroy(od_runtime* rt);
int od_rt_vp_count(const od_runtime* rt, int32_t* k);
int od_rt_proc_count(const od_runtime* rt, int32_t* p);
/* Engine::mapping                                        engine.hpp:163 */
int od_rt_mapping(const od_runtime* rt, int32_t* map /* K */);
/* Engine::subdomains                                     engine.hpp:161 */
int od_rt_subdomains(const od_runtime* rt, od_subdomain* out /* K */);
/* Engine::classify_vps                                 engine.hpp:281-287 */
int od_rt_classify(const od_runtime* rt, int32_t* classes /* K */);
/* Engine::load_field (current shifted field)            engine.hpp:165 */
int od_rt_load_field(const od_runtime* rt, double* c /* nx*ny */);
/*
 * Engine::step_time (engine.hpp:183-233), executed for real: one timestep of
 * halo exchange + Jacobi + physics over every resident chunk.  *wall is the
 * step's device time (max over ranks); samples[v] for every VP (gathered).
 */
int od_rt_step(od_runtime* rt, int32_t mode, int32_t epoch_step, int32_t global_step,
               double* wall, od_sample* samples /* K */);
/* Engine::run_epoch (engine.hpp:235-272) with real chunk migration */
int od_rt_run_epoch(od_runtime* rt, int32_t epoch_index, od_epoch_record* rec);
/*
 * Advance the epoch schedule by n timesteps (epoch boundaries perform
 * measurement, balancing and migration).  Records of completed epochs are not
 * returned; *epochs_done counts them.  Used by the benchmark.
 */
int od_rt_advance(od_runtime* rt, int32_t n_steps, int32_t* epochs_done);
/*
 * End-to-end variant of od_rt_advance for the host-facing path: every step
 * reads that step's load multiplier field (nx*ny doubles, [y][x]) from host
 * memory and writes the step's per-chunk device times (K doubles per step,
 * seconds; 0 for chunks on other ranks) to host_step_loads[step][vp].
 * host_c_fields: n_fields >= 1 caller fields; step i uses field min(i,
 * n_fields - 1) as its (already advected) load field.  NULL / n_fields = 0:
 * the runtime's own advected field crosses the host link each step.  The
 * runtime's advection schedule keeps advancing either way, so steps driven
 * afterwards by od_rt_advance continue it.  Both pointers must hold the sizes
 * above (the Python wrapper checks shape, dtype and contiguity).
 */
int od_rt_advance_host(od_runtime* rt, int32_t n_steps, const double* host_c_fields,
                       int32_t n_fields, double* host_step_loads /* n_steps*K */);
/* apply_plan plus the data movement of every moved chunk  cluster.hpp:130 */
int od_rt_migrate(od_runtime* rt, const od_move* moves, int32_t n_moves);
/*
 * Chunk state of VP vp if resident on this rank: u (fields*nz*h*w, layout
 * [f][k][y][x]) and a (nz*h*w, [k][y][x]).  *resident = 0 when not local.
 */
int od_rt_read_chunk(od_runtime* rt, int32_t vp, double* u, double* a,
                     int32_t* resident);
/* Diagnostics for the benchmark / roofline. */
typedef struct od_rt_stats {
  int64_t kernel_launches;     /* kernels of this library launched so far */
  int64_t steps;
  double jacobi_ms, physics_ms, pack_ms, exchange_ms; /* cumulative event time */
  int64_t jacobi_launches, physics_launches;
  int64_t halo_bytes_sent;     /* cumulative cross-rank halo bytes */
  int64_t migrated_bytes;      /* cumulative chunk bytes moved across ranks */
  int64_t physics_trips;       /* sum of trips of resident columns, last step */
  int32_t resident_chunks;
  int32_t pad_;
  int64_t jacobi_timed, physics_timed; /* launches whose event time is in *_ms */
  double fused_ms;
  int64_t fused_launches, fused_timed;
  int32_t last_kernel;         /* OD_KERNEL_* of the last step kernel launched */
  int32_t pad2_;
} od_rt_stats;
enum { OD_KERNEL_NONE = 0, OD_KERNEL_SEPARATE = 1, OD_KERNEL_STEP_GRID = 2,
       OD_KERNEL_STEP_WS = 3 };
int od_rt_stats_get(od_runtime* rt, od_rt_stats* out);
/* one row per completed epoch (od_rt_run_epoch, od_rt_advance, ..._host) */
typedef struct od_epoch_summary {
  int32_t epoch, strategy, n_moves, n_steps;
  double compute_total, migration_seconds, imbalance_before, imbalance_after;
  double boundary_seconds; /* host wall time of the epoch end: gather, decide, migrate */
} od_epoch_summary;
int od_rt_epoch_history(od_runtime* rt, od_epoch_summary* out, int32_t cap, int32_t* n);
/* enable per-kernel event timing (adds events around each batched kernel) */
int od_rt_set_profiling(od_runtime* rt, int32_t on);
int od_rt_synchronize(od_runtime* rt);
/*
 * Device wall time of individual steps by global step index (0 = the first
 * step this runtime ran): the wall Engine::step_time returns
 * (engine.hpp:183-233), i.e. for overlapped step kernels the interval between
 * consecutive step ends on the device clock.  out[i] = wall of step first+i in
 * seconds (max over ranks), NaN for steps whose epoch window has not been
 * collected yet.  Used by the benchmark to average exactly its timed steps.
 */
int od_rt_step_walls(od_runtime* rt, int64_t first, int32_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* OVERDECK_B200_H */
