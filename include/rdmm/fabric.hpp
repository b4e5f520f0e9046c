// rdmm/fabric.hpp -- the one-sided fabric API of the reference
// (/root/reference/proj/include/rdmm/fabric.hpp) over the B200 C-ABI.
//
// Same names and semantics: Fabric, FabricConfig, RankCtx, GlobalPtr,
// TrafficLog, Event, TileFetch, run_ranks.  What changed:
//  * heaps are device memory on each rank's GPU; every heap is mapped into
//    every rank's GPU so gets/puts are NVLink copies and kernels may load
//    peer data directly;
//  * get_nb is truly asynchronous (copy-engine copy on the rank's copy
//    stream; wait() makes the compute stream wait, the host does not block);
//  * fetch-add cells and queues live in a node-shared control segment;
//  * ranks may be threads of one process (run_ranks) or one process per GPU
//    (FabricConfig::first_local/nlocal/session);
//  * a rank failure aborts the fabric, so peers blocked in barrier() get a
//    fabric_error instead of the reference's deadlock (fabric.hpp:556-575).
#ifndef RDMM_B200_FABRIC_HPP
#define RDMM_B200_FABRIC_HPP

#include <cstddef>
#include <cstdint>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "rdmm/tile.hpp"

namespace rdmm {

using rank_t = std::uint32_t;

struct GlobalPtr {  // fabric.hpp:30-36
  rank_t rank = 0;
  std::uint64_t offset = 0;
  std::uint64_t length = 0;
  bool operator==(const GlobalPtr&) const = default;
  rdmm_gptr c() const { return rdmm_gptr{rank, 0, offset, length}; }
  static GlobalPtr of(const rdmm_gptr& g) { return {g.rank, g.offset, g.length}; }
};

struct Event {  // fabric.hpp:62-70
  enum class Kind { transfer, compute, queue_op };
  Kind kind;
  rank_t src = 0;
  rank_t dst = 0;
  std::uint64_t bytes = 0;
  std::uint64_t flops = 0;
};

struct TrafficCounters {  // fabric.hpp:72-87
  std::uint64_t bytes_put = 0, bytes_got = 0, puts = 0, gets = 0, atomic_ops = 0;
  TrafficCounters& operator+=(const TrafficCounters& o) {
    bytes_put += o.bytes_put;
    bytes_got += o.bytes_got;
    puts += o.puts;
    gets += o.gets;
    atomic_ops += o.atomic_ops;
    return *this;
  }
};

struct TileFetch {  // fabric.hpp:90-96
  rank_t src, dst;
  std::int64_t label;
  int matrix;
  std::uint32_t i, j;
};

// fabric.hpp:205-210 plus the B200 placement fields.
struct FabricConfig {
  rank_t nranks = 1;
  std::size_t heap_bytes = 64ull << 20;  // device heap per rank
  rank_t node_group = 6;
  std::size_t queue_capacity = 4096;
  // B200: GPU of each rank (default rank % device_count), the ranks hosted
  // by this process (default: all), the shm session shared by processes.
  std::vector<int> devices;
  rank_t first_local = 0;
  rank_t nlocal = 0;
  std::string session;
  std::size_t ctrl_bytes = 0;
};

class Fabric;

// Byte-exact accounting view (fabric.hpp:101-203).
class TrafficLog {
 public:
  explicit TrafficLog(Fabric* f) : f_(f) {}
  rank_t node_of(rank_t r) const;
  bool same_node(rank_t a, rank_t b) const { return node_of(a) == node_of(b); }
  TrafficCounters pair_total(rank_t src, rank_t dst) const;
  TrafficCounters total() const;
  std::vector<TileFetch> tile_fetches() const;
  void clear();

 private:
  Fabric* f_;
};

class Fabric {
 public:
  explicit Fabric(FabricConfig cfg) : cfg_(std::move(cfg)), traffic_(this) {
    if (cfg_.nranks == 0) throw fabric_error("nranks must be positive");
    if (cfg_.nlocal == 0) cfg_.nlocal = cfg_.nranks - cfg_.first_local;
    std::vector<int> dev(cfg_.nlocal);
    if (cfg_.devices.size() == cfg_.nlocal) {
      dev = cfg_.devices;
    } else if (cfg_.devices.size() == cfg_.nranks) {
      for (rank_t i = 0; i < cfg_.nlocal; ++i) dev[i] = cfg_.devices[cfg_.first_local + i];
    } else {
      int n = 1;
      rdmm_device_count(&n);
      for (rank_t i = 0; i < cfg_.nlocal; ++i) dev[i] = int((cfg_.first_local + i) % n);
    }
    rdmm_fabric_config c{};
    c.nranks = cfg_.nranks;
    c.node_group = cfg_.node_group;
    c.heap_bytes = cfg_.heap_bytes;
    c.queue_capacity = cfg_.queue_capacity;
    c.ctrl_bytes = cfg_.ctrl_bytes;
    c.first_local = cfg_.first_local;
    c.nlocal = cfg_.nlocal;
    c.devices = dev.data();
    c.session = cfg_.session.empty() ? nullptr : cfg_.session.c_str();
    check(rdmm_fabric_create(&c, &h_), "Fabric");
    devices_ = dev;
  }
  ~Fabric() { rdmm_fabric_destroy(h_); }
  Fabric(const Fabric&) = delete;
  Fabric& operator=(const Fabric&) = delete;

  rank_t nranks() const { return cfg_.nranks; }
  const FabricConfig& config() const { return cfg_; }
  TrafficLog& traffic() { return traffic_; }
  const TrafficLog& traffic() const { return traffic_; }
  rdmm_fabric* handle() const { return h_; }
  bool is_local(rank_t r) const { return r >= cfg_.first_local && r < cfg_.first_local + cfg_.nlocal; }
  rank_t first_local() const { return cfg_.first_local; }
  rank_t nlocal() const { return cfg_.nlocal; }
  int device_of(rank_t r) const { return devices_.at(r - cfg_.first_local); }

  GlobalPtr alloc(rank_t rank, std::size_t nbytes) {  // fabric.hpp:235-238
    rdmm_gptr g;
    std::uint64_t rem = 0;
    int rc = rdmm_heap_alloc(h_, rank, nbytes, &g);
    if (rc == RDMM_ERR_HEAP_EXHAUSTED) rdmm_heap_remaining(h_, rank, &rem);
    check(rc, "alloc", nbytes, rem);
    return GlobalPtr::of(g);
  }
  void free(GlobalPtr p) { check(rdmm_heap_free(h_, p.c()), "free"); }
  std::size_t heap_remaining(rank_t rank) const {
    std::uint64_t r = 0;
    check(rdmm_heap_remaining(h_, rank, &r), "heap_remaining");
    return r;
  }
  // Device address of p from `viewer`'s GPU (the reference's raw(), which
  // handed out host pointers, fabric.hpp:251-254).
  void* raw(GlobalPtr p, rank_t viewer) const {
    void* d = nullptr;
    check(rdmm_gptr_device(h_, viewer, p.c(), &d), "raw");
    return d;
  }
  void* raw(GlobalPtr p) const { return raw(p, is_local(p.rank) ? p.rank : cfg_.first_local); }
  // Host read of heap bytes bypassing traffic accounting (verification).
  void peek(GlobalPtr p, void* dst) const {
    check(rdmm_peek(h_, is_local(p.rank) ? p.rank : cfg_.first_local, p.c(), dst), "peek");
  }

  using queue_id = std::uint64_t;
  struct TransferHandle {  // fabric.hpp:256-259
    rdmm_handle h{nullptr, 0};
    bool waited = false;
    std::exception_ptr error;
  };

 private:
  FabricConfig cfg_;
  TrafficLog traffic_;
  rdmm_fabric* h_ = nullptr;
  std::vector<int> devices_;
};

inline rank_t TrafficLog::node_of(rank_t r) const {
  rank_t g = f_->config().node_group;
  return r / (g ? g : 1);
}
inline TrafficCounters TrafficLog::pair_total(rank_t s, rank_t d) const {
  rdmm_traffic t;
  rdmm_traffic_pair(f_->handle(), s, d, &t);
  return {t.bytes_put, t.bytes_got, t.puts, t.gets, t.atomic_ops};
}
inline TrafficCounters TrafficLog::total() const {
  rdmm_traffic t;
  rdmm_traffic_total(f_->handle(), &t);
  return {t.bytes_put, t.bytes_got, t.puts, t.gets, t.atomic_ops};
}
inline std::vector<TileFetch> TrafficLog::tile_fetches() const {
  const std::uint64_t n = rdmm_tile_fetches(f_->handle(), nullptr, 0);
  std::vector<rdmm_tile_fetch> raw(n);
  rdmm_tile_fetches(f_->handle(), raw.data(), n);
  std::vector<TileFetch> out;
  out.reserve(n);
  for (auto& r : raw) out.push_back({r.src, r.dst, r.label, r.matrix, r.i, r.j});
  return out;
}
inline void TrafficLog::clear() { rdmm_traffic_clear(f_->handle()); }

// Per-rank handle through which all fabric operations are issued
// (fabric.hpp:416-552).
class RankCtx {
 public:
  RankCtx(Fabric& f, rank_t rank) : fabric_(&f), rank_(rank) {}

  rank_t rank() const { return rank_; }
  rank_t nranks() const { return fabric_->nranks(); }
  Fabric& fabric() { return *fabric_; }
  rdmm_fabric* h() const { return fabric_->handle(); }
  int device() const { return fabric_->device_of(rank_); }
  // 0: compute stream, 1/2: copy streams
  rdmm_stream_t stream(int which = 0) const { return rdmm_fabric_stream(h(), rank_, which); }

  void set_phase(std::int64_t label) { rdmm_set_phase(h(), rank_, label); }
  std::int64_t phase() const { return rdmm_phase(h(), rank_); }

  // Events accumulate inside the fabric; flush_events() appends them here.
  void set_event_sink(std::vector<Event>* sink) {
    sink_ = sink;
    rdmm_event_sink(h(), rank_, sink ? 1 : 0);
  }
  void flush_events() {
    if (!sink_) return;
    const std::uint64_t n = rdmm_events(h(), rank_, nullptr, 0);
    std::vector<rdmm_event> ev(n);
    rdmm_events(h(), rank_, ev.data(), n);
    for (auto& e : ev)
      sink_->push_back({static_cast<Event::Kind>(e.kind), e.src, e.dst, e.bytes, e.flops});
    rdmm_event_sink(h(), rank_, 1);  // clears the fabric-side buffer
  }

  GlobalPtr alloc(std::size_t nbytes) { return fabric_->alloc(rank_, nbytes); }
  GlobalPtr alloc_on(rank_t r, std::size_t nbytes) { return fabric_->alloc(r, nbytes); }
  void free(GlobalPtr p) { fabric_->free(p); }

  // Host-buffer one-sided transfers (fabric.hpp:436-454).
  void put(std::span<const std::byte> src, GlobalPtr dst) {
    if (src.size() != dst.length)
      throw fabric_error("put: span length does not match pointer length");
    check(rdmm_put_host(h(), rank_, src.data(), dst.c()), "put");
  }
  void get(GlobalPtr src, std::span<std::byte> dst) {
    if (dst.size() != src.length)
      throw fabric_error("get: span length does not match pointer length");
    check(rdmm_get_host(h(), rank_, src.c(), dst.data()), "get");
  }
  // Device-buffer non-blocking get (fabric.hpp:456-464), asynchronous.
  Fabric::TransferHandle get_nb(GlobalPtr src, void* dev_dst, int copy_stream = 1) {
    Fabric::TransferHandle t;
    int rc = rdmm_get_nb(h(), rank_, src.c(), dev_dst, stream(copy_stream), &t.h);
    if (rc) {
      try {
        check(rc, "get_nb");
      } catch (...) {
        t.error = std::current_exception();
      }
    }
    return t;
  }
  // Idempotent; makes `consumer` (default: the compute stream) wait for the
  // transfer without blocking the host (fabric.hpp:467-471).
  void wait(Fabric::TransferHandle& t, rdmm_stream_t consumer = nullptr) {
    if (t.waited) return;
    t.waited = true;
    if (t.error) std::rethrow_exception(t.error);
    check(rdmm_wait(h(), &t.h, consumer ? consumer : stream(0)), "wait");
  }

  std::int64_t fetch_add(GlobalPtr counter, std::int64_t delta) {  // fabric.hpp:473-487
    std::int64_t old = 0;
    check(rdmm_fetch_add_i64(h(), rank_, counter.c(), delta, &old), "fetch_add");
    return old;
  }
  void put_i64(std::int64_t v, GlobalPtr dst) {
    put(std::as_bytes(std::span{&v, 1}), dst);
  }
  std::int64_t get_i64(GlobalPtr src) {
    std::int64_t v = 0;
    get(src, std::as_writable_bytes(std::span{&v, 1}));
    return v;
  }

  // Queues (fabric.hpp:502-528) with an inline header of <= 40 bytes.
  void queue_push(Fabric::queue_id q, GlobalPtr v, const void* inl = nullptr,
                  std::uint32_t inl_bytes = 0) {
    check(rdmm_queue_push(h(), rank_, q, v.c(), inl, inl_bytes), "queue_push");
  }
  std::optional<GlobalPtr> queue_pop(Fabric::queue_id q, void* inl = nullptr,
                                     std::uint32_t inl_bytes = 0) {
    rdmm_gptr g;
    int got = 0;
    check(rdmm_queue_pop(h(), rank_, q, &g, inl, inl_bytes, &got), "queue_pop");
    if (!got) return std::nullopt;
    return GlobalPtr::of(g);
  }

  // Collective; device work issued on this rank's fabric streams before the
  // barrier is complete after it (fabric.hpp:530-532).
  void barrier() { check(rdmm_barrier(h(), rank_), "barrier"); }

  void record_tile_fetch(rank_t owner, int matrix, std::uint32_t i, std::uint32_t j) {
    rdmm_record_tile_fetch(h(), rank_, owner, matrix, i, j);
  }
  void emit_compute(std::uint64_t flops) { rdmm_emit_compute(h(), rank_, flops); }

 private:
  Fabric* fabric_;
  rank_t rank_;
  std::vector<Event>* sink_ = nullptr;
};

// Runs fn(ctx) for every rank hosted by this process, one thread per rank
// (fabric.hpp:556-575).  A failing rank aborts the fabric so peers blocked in
// a barrier return instead of deadlocking; the first error is rethrown.
template <typename F>
void run_ranks(Fabric& f, F&& fn) {
  if (f.nlocal() == 1) {
    // one rank in this process (one process per GPU): run it on the calling
    // thread -- no thread start per collective call -- and restore the
    // caller's current device afterwards
    int prev = 0;
    const bool have_prev = rdmm_get_device(&prev) == RDMM_OK;
    const rank_t r = f.first_local();
    try {
      rdmm_set_device(f.device_of(r));
      RankCtx ctx(f, r);
      fn(ctx);
    } catch (const std::exception& e) {
      rdmm_fabric_abort(f.handle(), e.what());
      if (have_prev) rdmm_set_device(prev);
      throw;
    } catch (...) {
      rdmm_fabric_abort(f.handle(), "rank failed");
      if (have_prev) rdmm_set_device(prev);
      throw;
    }
    if (have_prev) rdmm_set_device(prev);
    return;
  }
  std::vector<std::thread> threads;
  std::mutex err_mu;
  std::exception_ptr first_error;
  for (rank_t r = f.first_local(); r < f.first_local() + f.nlocal(); ++r) {
    threads.emplace_back([&, r] {
      try {
        rdmm_set_device(f.device_of(r));
        RankCtx ctx(f, r);
        fn(ctx);
      } catch (const std::exception& e) {
        rdmm_fabric_abort(f.handle(), e.what());
        std::scoped_lock lk(err_mu);
        if (!first_error) first_error = std::current_exception();
      } catch (...) {
        rdmm_fabric_abort(f.handle(), "rank failed");
        std::scoped_lock lk(err_mu);
        if (!first_error) first_error = std::current_exception();
      }
    });
  }
  for (auto& t : threads) t.join();
  if (first_error) std::rethrow_exception(first_error);
}

}  // namespace rdmm

#endif  // RDMM_B200_FABRIC_HPP
