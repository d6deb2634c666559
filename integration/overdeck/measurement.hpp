#pragma once
// Drop-in replacement of the reference's overdeck/measurement.hpp
// (/root/reference/proj/include/overdeck/measurement.hpp:1-99): the per-VP load
// database of the paper's measurement protocol, served by libod_b200's
// od_loaddb_* (include/overdeck_b200.h), with the reference's names, value
// types and exception behaviour.
//
//   StepSample, MeasurementWindow   measurement.hpp:14-37 (value types)
//   LoadDB                          measurement.hpp:40-69 -> od_loaddb_create/record/clear
//   record_step, epoch_loads        measurement.hpp:72-91 -> od_loaddb_record/epoch_loads
//   launch_only_sample              measurement.hpp:95-97
#include <memory>
#include <string>
#include <vector>

#include "overdeck/cluster.hpp"
#include "overdeck/errors.hpp"
#include "overdeck/gpu_cost.hpp"
#include "overdeck_b200.h"

namespace overdeck {

namespace b200 {
inline void check_db(int rc) {
  if (rc == OD_OK) return;
  const std::string msg = od_last_error();
  if (rc == OD_EVALIDATION) throw ValidationError(msg);
  throw RuntimeFault(msg);
}
}  // namespace b200

struct StepSample {
  VpId vp = 0;
  int step = 0;  // 0-based within the epoch
  LaunchMode mode = LaunchMode::Sync;
  double value = 0.0;  // seconds
};

struct MeasurementWindow {
  int async_steps = 0;
  int sync_steps = 1;

  int epoch_steps() const { return async_steps + sync_steps; }
  void validate() const {
    if (async_steps < 0) throw ValidationError("window.async_steps must be >= 0");
    if (sync_steps < 1) throw ValidationError("window.sync_steps must be >= 1");
  }
  LaunchMode mode_of_step(int step) const {
    return step < async_steps ? LaunchMode::Async : LaunchMode::Sync;
  }
};

class LoadDB {
 public:
  explicit LoadDB(int vp_count, MeasurementWindow window) : vp_count_(vp_count), window_(window) {
    od_loaddb* h = nullptr;
    b200::check_db(od_loaddb_create(vp_count, window.async_steps, window.sync_steps, &h));
    db_.reset(h, od_loaddb_destroy);
  }

  int vp_count() const { return vp_count_; }
  const MeasurementWindow& window() const { return window_; }
  const std::vector<StepSample>& samples() const { return samples_; }

  void record(const StepSample& s) {
    const od_sample c{s.vp, s.step, s.mode == LaunchMode::Async ? OD_ASYNC : OD_SYNC, 0, s.value};
    b200::check_db(od_loaddb_record(db_.get(), &c));
    samples_.push_back(s);
  }
  void clear() {
    b200::check_db(od_loaddb_clear(db_.get()));
    samples_.clear();
  }
  const od_loaddb* handle() const { return db_.get(); }

 private:
  int vp_count_ = 0;
  MeasurementWindow window_;
  std::shared_ptr<od_loaddb> db_;
  std::vector<StepSample> samples_;  // (the reference's samples() view)
};

inline void record_step(LoadDB& db, const StepSample& sample) { db.record(sample); }

inline LoadVector epoch_loads(const LoadDB& db) {
  LoadVector out(static_cast<size_t>(db.vp_count()), 0.0);
  b200::check_db(od_loaddb_epoch_loads(db.handle(), out.data()));
  return out;
}

inline StepSample launch_only_sample(VpId vp, int step, const GpuModel& gpu) {
  return {vp, step, LaunchMode::Async, gpu.launch_overhead};
}

}  // namespace overdeck
