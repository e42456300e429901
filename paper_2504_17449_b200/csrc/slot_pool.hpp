// SPDX-License-Identifier: Apache-2.0
//
// SlotPool — the HBM adapter slot pool's residency policy.
//
// Restates DeviceSlotPool (proj/include/hmi/adapters/device_pool.hpp:40-98,
// proj/src/adapters/device_pool.cpp:14-217) decision for decision, keyed by a
// dense task index instead of the task-id string:
//   * residency per (task, layer) under a byte budget in the reference's f32
//     accounting (adapter_set.hpp:24-27), so LRU decisions and LoadRecords are
//     identical to the reference's for the same capacity and access trace;
//   * eviction of whole tasks, least-recently-used `last_used` tick first,
//     skipping protected (same-call) and pinned tasks (make_room, :14-48);
//   * ensure_resident throws CapacityError (:50-91); try_ensure_layer_resident
//     returns nullopt when only pinned tasks block (:93-136).
// In addition every resident (task, layer) owns one physical slot of the HBM
// arena; slots are recycled from evicted tasks. This is the part the GPU adds.
// Placement prefers blocks: the arena's first (slots / block_len) * block_len slots form
// blocks of block_len (= the model's layer count); a task claims a free block with its
// first resident layer and its layer l then goes to slot block * block_len + l, so a
// whole-task miss is one contiguous host -> HBM copy. Any free slot is used when no
// block is free (the byte budget, not the placement, decides residency).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <vector>

namespace hmi_b200 {

struct PoolLoad {
  uint32_t layer;
  int32_t slot;
};

struct PoolFree {
  uint32_t task, layer;
  int32_t slot;
};

// LoadRecord (device_pool.hpp:27-33) + the physical placement.
struct PoolRecord {
  uint32_t task = 0;
  bool hit = false;
  uint64_t bytes = 0;
  std::vector<uint32_t> evicted;        // whole tasks evicted, in eviction order
  std::vector<PoolLoad> loads;          // (layer, slot) made resident by this record
  std::vector<PoolFree> freed;     // (task, layer, slot) released by evictions
};

class SlotPool {
 public:
  SlotPool(uint64_t capacity_bytes, uint32_t physical_slots, uint32_t block_len = 1);

  // AdapterStore registration mirror: a task's layer count and per-layer bytes.
  void set_task(uint32_t task, uint32_t layers, uint64_t layer_bytes);
  bool has_task(uint32_t task) const { return tasks_.count(task) != 0; }
  void remove_task(uint32_t task, std::vector<PoolFree>* freed);

  std::vector<PoolRecord> ensure_resident(const std::vector<uint32_t>& task_ids);
  std::optional<std::vector<PoolRecord>> try_ensure_layer_resident(
      const std::vector<uint32_t>& task_ids, uint32_t layer);

  void pin(const std::vector<uint32_t>& task_ids);
  void unpin(const std::vector<uint32_t>& task_ids);
  void touch(const std::vector<uint32_t>& task_ids);
  bool evict(uint32_t task, std::vector<PoolFree>* freed);

  int32_t slot_of(uint32_t task, uint32_t layer) const;
  bool is_layer_resident(uint32_t task, uint32_t layer) const;
  uint32_t layers_of(uint32_t task) const;

  uint64_t capacity_bytes() const { return capacity_; }
  uint64_t resident_bytes() const { return resident_bytes_; }
  uint64_t max_resident_bytes_seen() const { return max_resident_bytes_; }
  uint64_t resident_task_count() const;
  uint64_t hits() const { return hits_; }
  uint64_t loads() const { return loads_; }
  uint32_t physical_slots() const { return static_cast<uint32_t>(n_slots_); }

  // Decisions a failed call made before it failed: ensure_resident throwing CapacityError,
  // try_ensure_layer_resident returning nullopt. The reference mutates its state as it goes
  // and keeps those decisions (device_pool.cpp:50-136): the records of the tasks placed
  // before the failure (loads) and the evictions of the failing task (freed only). A caller
  // that retries must act on them (copy the loads, ship the slot-table deltas) — the retry
  // sees those tasks as hits.
  std::vector<PoolRecord> take_partial() {
    std::vector<PoolRecord> v;
    v.swap(partial_);
    return v;
  }

  // Rolls back one (task, layer) placement whose copy was never issued: the layer is no
  // longer resident and its slot is free again (a failed submit undoing its own decisions).
  void unload(uint32_t task, uint32_t layer);

 private:
  std::vector<PoolRecord> partial_;
  struct Residency {
    std::map<uint32_t, int32_t> layers;  // layer -> physical slot
    uint64_t bytes = 0;
    uint64_t last_used = 0;
    uint32_t pins = 0;
  };
  struct TaskInfo {
    uint32_t layers;
    uint64_t layer_bytes;
  };

  void stash_partial(std::vector<PoolRecord>& done, PoolRecord& failing);
  bool make_room(uint64_t needed, const std::set<uint32_t>& protect, PoolRecord& rec);
  void release(uint32_t task, Residency& r, std::vector<PoolFree>* freed);
  int32_t take_slot(uint32_t task, uint32_t layer);
  void free_slot(int32_t slot);
  void drop_claim(uint32_t task);

  uint64_t capacity_;
  size_t n_slots_;
  uint32_t block_len_;
  int32_t n_blocks_;                    // full blocks; slots >= n_blocks_ * block_len_ are loose
  std::vector<uint8_t> slot_free_;
  std::vector<uint32_t> block_free_;    // free slots per block
  std::vector<int64_t> block_owner_;    // claiming task, or -1
  std::map<uint32_t, int32_t> claim_;   // task -> claimed block
  std::set<int32_t> free_blocks_;       // fully free, unclaimed blocks
  std::set<int32_t> loose_free_;        // free slots usable when no block is free
  size_t n_free_ = 0;
  std::map<uint32_t, TaskInfo> tasks_;
  std::map<uint32_t, Residency> resident_;
  // (last_used, task) of every resident record: the reference scans all residents for the
  // minimum last_used (device_pool.cpp:25-35); ticks are unique, so walking this ordered
  // index from the front and skipping protected / pinned records picks the same victim
  // in O(k log n) instead of O(n).
  std::set<std::pair<uint64_t, uint32_t>> lru_;
  void set_last_used(uint32_t task, Residency& r, uint64_t tick);
  void forget(uint32_t task, const Residency& r) { lru_.erase({r.last_used, task}); }
  uint64_t resident_bytes_ = 0;
  uint64_t max_resident_bytes_ = 0;
  uint64_t tick_ = 0;
  uint64_t hits_ = 0;
  uint64_t loads_ = 0;
};

}  // namespace hmi_b200
