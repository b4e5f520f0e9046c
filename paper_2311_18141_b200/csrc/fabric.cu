// fabric.cu -- the one-sided fabric of the reference (fabric.hpp) rebuilt
// for one B200 box: device heaps mapped into every rank's GPU (peer access /
// CUDA IPC over NVLink 5), a node-shared control segment for atomics, queues
// and the barrier, copy-engine get/put on per-rank streams, and the
// byte-exact traffic log (fabric.hpp:98-203).  See include/rdmm_cuda.h.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace rdmm_impl {
namespace {

constexpr uint32_t kMaxRanks = 64;
constexpr uint32_t kMaxColl = 1024;
constexpr uint64_t kMagic = 0x31424146'4d4d4452ull;  // "RDMMFAB1"
constexpr uint32_t kInline = 40;

struct alignas(64) QueueSlot {
  std::atomic<uint32_t> ready;
  uint32_t inl_bytes;
  rdmm_gptr v;
  uint8_t inl[kInline];
};

struct alignas(64) QueueHdr {
  alignas(64) std::atomic<int64_t> tail;  // reserved by producers
  alignas(64) std::atomic<int64_t> head;  // consumed by the owner
  uint64_t capacity;
  uint32_t owner;
};

struct CollEntry {
  uint64_t tag;
  uint64_t offset;  // in the arena
  uint64_t bytes;
  uint32_t releases;
  uint32_t live;
};

struct RankSlot {
  cudaIpcMemHandle_t heap;
  uint64_t heap_bytes;
  int32_t device;
  int32_t pid;
  std::atomic<uint32_t> published;
};

struct Ctrl {
  uint64_t magic;
  uint32_t nranks;
  std::atomic<uint32_t> ready;
  alignas(64) std::atomic<uint32_t> bar_count;
  alignas(64) std::atomic<uint32_t> bar_gen;
  alignas(64) std::atomic<uint32_t> lock;
  uint64_t arena_used;
  uint64_t arena_size;
  uint32_t ncoll;
  alignas(64) std::atomic<uint32_t> abort;
  char abort_msg[256];
  RankSlot ranks[kMaxRanks];
  CollEntry coll[kMaxColl];
};

constexpr size_t ctrl_header_bytes() {
  return (sizeof(Ctrl) + 4095) & ~size_t(4095);
}

struct SpinLock {
  std::atomic<uint32_t>& a;
  explicit SpinLock(std::atomic<uint32_t>& x) : a(x) {
    uint32_t exp = 0;
    int n = 0;
    while (!a.compare_exchange_weak(exp, 1, std::memory_order_acquire)) {
      exp = 0;
      if (++n > 64) std::this_thread::yield();
    }
  }
  ~SpinLock() { a.store(0, std::memory_order_release); }
};

struct Heap {
  char* base = nullptr;
  uint64_t cap = 0;
  uint64_t remaining = 0;
  std::vector<std::pair<uint64_t, uint64_t>> free_list;  // (offset, size)
  std::map<uint64_t, uint64_t> live;                     // offset -> size
  mutable std::mutex mu;

  static uint64_t align_up(uint64_t n) { return n == 0 ? 8 : (n + 7) & ~7ull; }

  // fabric.hpp:284-303 first fit, 8-byte granules; requests of >= 256
  // bytes are additionally placed on 256-byte boundaries so device tiles
  // keep the 16-byte alignment the vectorised kernels need (padding stays
  // free and is reused by small requests).
  bool alloc(uint64_t nbytes, uint64_t* off) {
    std::lock_guard<std::mutex> lk(mu);
    const uint64_t need = align_up(nbytes);
    const uint64_t align = need >= 256 ? 256 : 8;
    for (std::size_t b = 0; b < free_list.size(); ++b) {
      const uint64_t bo = free_list[b].first, bs = free_list[b].second;
      const uint64_t start = (bo + align - 1) & ~(align - 1);
      const uint64_t pad = start - bo;
      if (bs < pad + need) continue;
      free_list.erase(free_list.begin() + std::ptrdiff_t(b));
      if (pad) free_list.push_back({bo, pad});
      if (bs > pad + need) free_list.push_back({start + need, bs - pad - need});
      std::sort(free_list.begin(), free_list.end());
      *off = start;
      live[start] = need;
      remaining -= need;
      return true;
    }
    return false;
  }
  // fabric.hpp:305-314
  bool release(uint64_t off) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = live.find(off);
    if (it == live.end()) return false;
    remaining += it->second;
    free_list.push_back({it->first, it->second});
    live.erase(it);
    std::sort(free_list.begin(), free_list.end());
    std::vector<std::pair<uint64_t, uint64_t>> merged;
    for (auto& b : free_list) {
      if (!merged.empty() && merged.back().first + merged.back().second == b.first)
        merged.back().second += b.second;
      else
        merged.push_back(b);
    }
    free_list.swap(merged);
    return true;
  }
  // fabric.hpp:316-328
  bool valid(uint64_t off, uint64_t len) const {
    std::lock_guard<std::mutex> lk(mu);
    auto it = live.upper_bound(off);
    if (it != live.begin()) {
      --it;
      if (off >= it->first && off + len <= it->first + it->second) return true;
    }
    return len == 0 && off <= cap;
  }
};

struct Local {
  uint32_t rank = 0;
  int device = 0;
  Heap heap;
  // 0 compute, 1-2 copy engines, 3 side compute (concat of pipelined fetches)
  cudaStream_t streams[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t label = 0;
  bool sink = false;
  std::vector<rdmm_event> events;
  unsigned long long* atomic_slot = nullptr;  // pinned, device-space fetch_add
  cudaStream_t atomic_stream = nullptr;       // idle stream for device fetch_add
};

using TKey = std::tuple<uint32_t, uint32_t, int64_t>;

__global__ void k_fetch_add(unsigned long long* cell, long long delta,
                            unsigned long long* out) {
  *out = atomicAdd(cell, static_cast<unsigned long long>(delta));
}

}  // namespace
}  // namespace rdmm_impl

using namespace rdmm_impl;

struct rdmm_fabric {
  rdmm_fabric_config cfg{};
  std::string session;
  bool owns_shm = false, shared = false;
  Ctrl* ctrl = nullptr;
  size_t ctrl_map_bytes = 0;
  char* arena = nullptr;
  std::vector<std::unique_ptr<Local>> locals;
  // base[local index][rank]: device address of rank's heap on that GPU
  std::vector<std::vector<char*>> base;
  std::vector<uint64_t> heap_bytes;  // per rank
  std::vector<std::pair<int, void*>> ipc_opened;
  std::atomic<uint64_t> uid{0};
  mutable std::mutex tmu;
  std::map<TKey, rdmm_traffic> cells;
  std::vector<rdmm_tile_fetch> fetches;

  Local* local(uint32_t r) {
    if (r < cfg.first_local || r >= cfg.first_local + cfg.nlocal) return nullptr;
    return locals[r - cfg.first_local].get();
  }
  bool same_node(uint32_t a, uint32_t b) const {
    const uint32_t g = cfg.node_group ? cfg.node_group : 1;
    return a / g == b / g;
  }
  void emit(Local* L, int kind, uint32_t src, uint32_t dst, uint64_t bytes,
            uint64_t flops) {
    if (L && L->sink) L->events.push_back({kind, src, dst, bytes, flops});
  }
  void record_get(uint32_t owner, uint32_t caller, uint64_t bytes) {
    Local* L = local(caller);
    {
      std::lock_guard<std::mutex> lk(tmu);
      auto& c = cells[TKey{owner, caller, L ? L->label : 0}];
      c.bytes_got += bytes;
      c.gets += 1;
    }
    emit(L, 0, owner, caller, bytes, 0);
  }
  void record_put(uint32_t caller, uint32_t dst, uint64_t bytes) {
    Local* L = local(caller);
    {
      std::lock_guard<std::mutex> lk(tmu);
      auto& c = cells[TKey{caller, dst, L ? L->label : 0}];
      c.bytes_put += bytes;
      c.puts += 1;
    }
    emit(L, 0, caller, dst, bytes, 0);
  }
  void record_atomic(uint32_t caller, uint32_t owner) {
    Local* L = local(caller);
    std::lock_guard<std::mutex> lk(tmu);
    cells[TKey{caller, owner, L ? L->label : 0}].atomic_ops += 1;
  }
};

namespace {

int check_gptr(rdmm_fabric* f, rdmm_gptr p, bool ctrl_ok) {
  if (p.rank >= f->cfg.nranks)
    return fail(RDMM_ERR_FABRIC, "rank out of range");
  if (p.offset & RDMM_CTRL_BIT) {
    if (!ctrl_ok) return fail(RDMM_ERR_FABRIC, "control cell used as heap data");
    const uint64_t off = p.offset & ~RDMM_CTRL_BIT;
    if (off + p.length > f->ctrl->arena_size)
      return fail(RDMM_ERR_FABRIC, "dangling or out-of-range global pointer");
    return RDMM_OK;
  }
  Local* owner = f->local(p.rank);
  if (owner) {
    if (!owner->heap.valid(p.offset, p.length))
      return fail(RDMM_ERR_FABRIC, "dangling or out-of-range global pointer");
  } else if (p.offset + p.length > f->heap_bytes[p.rank]) {
    return fail(RDMM_ERR_FABRIC, "dangling or out-of-range global pointer");
  }
  return RDMM_OK;
}

char* dev_addr(rdmm_fabric* f, Local* caller, rdmm_gptr p) {
  return f->base[caller->rank - f->cfg.first_local][p.rank] + p.offset;
}

int wait_all_published(rdmm_fabric* f) {
  for (uint32_t r = 0; r < f->cfg.nranks; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    while (f->ctrl->ranks[r].published.load(std::memory_order_acquire) == 0) {
      if (f->ctrl->abort.load()) return fail(RDMM_ERR_FABRIC, "fabric aborted");
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
        return fail(RDMM_ERR_FABRIC, "timeout waiting for peer ranks");
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  return RDMM_OK;
}

uint64_t coll_alloc(rdmm_fabric* f, uint64_t tag, uint64_t bytes, bool* fresh) {
  Ctrl* c = f->ctrl;
  SpinLock lk(c->lock);
  for (uint32_t i = 0; i < c->ncoll; ++i)
    if (c->coll[i].live && c->coll[i].tag == tag) {
      *fresh = false;
      return c->coll[i].offset;
    }
  const uint64_t need = (bytes + 127) & ~127ull;
  if (c->ncoll >= kMaxColl || c->arena_used + need > c->arena_size) return ~0ull;
  CollEntry& e = c->coll[c->ncoll++];
  e.tag = tag;
  e.offset = c->arena_used;
  e.bytes = need;
  e.releases = 0;
  e.live = 1;
  c->arena_used += need;
  std::memset(f->arena + e.offset, 0, need);
  *fresh = true;
  return e.offset;
}

// Sense-free generation barrier over all P ranks; `n` arrivals at once (a
// process arriving for all of its local ranks during setup).
int barrier_n(rdmm_fabric* f, uint32_t n) {
  Ctrl* c = f->ctrl;
  const uint32_t gen = c->bar_gen.load(std::memory_order_acquire);
  if (c->bar_count.fetch_add(n, std::memory_order_acq_rel) + n == c->nranks) {
    c->bar_count.store(0, std::memory_order_relaxed);
    c->bar_gen.fetch_add(1, std::memory_order_acq_rel);
    return RDMM_OK;
  }
  int spins = 0;
  while (c->bar_gen.load(std::memory_order_acquire) == gen) {
    if (c->abort.load(std::memory_order_acquire))
      return fail(RDMM_ERR_FABRIC, std::string("fabric aborted: ") + c->abort_msg);
    if (++spins < 2000) {
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    } else if (spins < 20000) {
      std::this_thread::yield();
    } else {
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
  return RDMM_OK;
}

}  // namespace

extern "C" int rdmm_fabric_create(const rdmm_fabric_config* cfg,
                                  rdmm_fabric** out) {
  *out = nullptr;
  if (!cfg || cfg->nranks == 0)
    return fail(RDMM_ERR_FABRIC, "nranks must be positive");
  if (cfg->nranks > kMaxRanks)
    return fail(RDMM_ERR_FABRIC, "nranks exceeds 64");
  if (cfg->nlocal == 0 || cfg->first_local + cfg->nlocal > cfg->nranks)
    return fail(RDMM_ERR_FABRIC, "bad local rank range");
  // Every error return below runs the deleter: the abort flag releases peers
  // waiting in wait_all_published / barrier_n, and destroy unlinks the shm
  // name and frees the heaps, streams and IPC mappings created so far.
  struct Cleanup {
    void operator()(rdmm_fabric* p) const {
      rdmm_fabric_abort(p, "fabric creation failed");
      rdmm_fabric_destroy(p);
    }
  };
  std::unique_ptr<rdmm_fabric, Cleanup> f(new rdmm_fabric());
  f->cfg = *cfg;
  f->cfg.devices = nullptr;
  f->cfg.session = nullptr;
  if (f->cfg.queue_capacity == 0) f->cfg.queue_capacity = 4096;
  if (f->cfg.node_group == 0) f->cfg.node_group = 6;
  const uint64_t arena = cfg->ctrl_bytes ? cfg->ctrl_bytes : (64ull << 20);
  f->shared = cfg->session && cfg->session[0];
  if (!f->shared && cfg->nlocal != cfg->nranks)
    return fail(RDMM_ERR_FABRIC, "a session name is required for multi-process fabrics");
  // ---------------- control segment
  f->ctrl_map_bytes = ctrl_header_bytes() + arena;
  void* mem = nullptr;
  if (f->shared) {
    f->session = std::string("/rdmm_") + cfg->session;
    int fd = shm_open(f->session.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd >= 0) {
      f->owns_shm = true;
      if (ftruncate(fd, off_t(f->ctrl_map_bytes)) != 0) {
        close(fd);
        shm_unlink(f->session.c_str());
        return fail(RDMM_ERR_FABRIC, "ftruncate of control segment failed");
      }
    } else {
      auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        fd = shm_open(f->session.c_str(), O_RDWR, 0600);
        if (fd >= 0) {
          struct stat st;
          if (fstat(fd, &st) == 0 && uint64_t(st.st_size) >= f->ctrl_map_bytes) break;
          close(fd);
        }
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          return fail(RDMM_ERR_FABRIC, "cannot attach control segment " + f->session);
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    mem = mmap(nullptr, f->ctrl_map_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (mem == MAP_FAILED) return fail(RDMM_ERR_FABRIC, "mmap of control segment failed");
  } else {
    mem = mmap(nullptr, f->ctrl_map_bytes, PROT_READ | PROT_WRITE,
               MAP_SHARED | MAP_ANONYMOUS, -1, 0);
    if (mem == MAP_FAILED) return fail(RDMM_ERR_FABRIC, "mmap of control segment failed");
    f->owns_shm = true;
  }
  f->ctrl = static_cast<Ctrl*>(mem);
  f->arena = static_cast<char*>(mem) + ctrl_header_bytes();
  if (f->owns_shm) {
    Ctrl* c = f->ctrl;
    c->nranks = cfg->nranks;
    c->arena_size = arena;
    c->arena_used = 0;
    c->ncoll = 0;
    c->magic = kMagic;
    c->ready.store(1, std::memory_order_release);
  } else {
    auto t0 = std::chrono::steady_clock::now();
    while (f->ctrl->ready.load(std::memory_order_acquire) == 0) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        return fail(RDMM_ERR_FABRIC, "control segment never became ready");
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (f->ctrl->magic != kMagic || f->ctrl->nranks != cfg->nranks)
      return fail(RDMM_ERR_FABRIC, "control segment belongs to another fabric");
  }
  // pinned + device-mapped so kernels may observe control cells too
  // (skipped for control-plane-only fabrics: every local device < 0)
  bool any_gpu = false;
  for (uint32_t i = 0; i < cfg->nlocal; ++i)
    any_gpu |= !cfg->devices || cfg->devices[i] >= 0;
  if (any_gpu) {
    cudaHostRegister(mem, f->ctrl_map_bytes, cudaHostRegisterPortable);
    cudaGetLastError();
  }
  // ---------------- local ranks: heaps, streams
  for (uint32_t i = 0; i < cfg->nlocal; ++i) {
    auto L = std::make_unique<Local>();
    L->rank = cfg->first_local + i;
    L->device = cfg->devices ? cfg->devices[i] : 0;
    if (L->device < 0) {
      // control-plane-only rank (no GPU): cells, queues, barrier, no heap
      if (cfg->heap_bytes)
        return fail(RDMM_ERR_FABRIC, "a rank without a device cannot have a heap");
      RankSlot& rs = f->ctrl->ranks[L->rank];
      rs.heap_bytes = 0;
      rs.device = -1;
      rs.pid = int32_t(getpid());
      rs.published.store(1, std::memory_order_release);
      f->locals.push_back(std::move(L));
      continue;
    }
    RDMM_CUDA_TRY(cudaSetDevice(L->device));
    void* hp = nullptr;
    RDMM_CUDA_TRY(cudaMalloc(&hp, cfg->heap_bytes ? cfg->heap_bytes : 8));
    RDMM_CUDA_TRY(cudaMemset(hp, 0, cfg->heap_bytes ? cfg->heap_bytes : 8));
    L->heap.base = static_cast<char*>(hp);
    L->heap.cap = cfg->heap_bytes;
    L->heap.remaining = cfg->heap_bytes;
    if (cfg->heap_bytes) L->heap.free_list.push_back({0, cfg->heap_bytes});
    for (auto& s : L->streams)
      RDMM_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    RDMM_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&L->atomic_slot), 64,
                                cudaHostAllocPortable));
    RDMM_CUDA_TRY(cudaStreamCreateWithFlags(&L->atomic_stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, L->device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    RankSlot& rs = f->ctrl->ranks[L->rank];
    rs.heap_bytes = cfg->heap_bytes;
    rs.device = L->device;
    rs.pid = int32_t(getpid());
    if (f->shared) RDMM_CUDA_TRY(cudaIpcGetMemHandle(&rs.heap, hp));
    rs.published.store(1, std::memory_order_release);
    f->locals.push_back(std::move(L));
  }
  if (int rc = wait_all_published(f.get())) return rc;
  f->heap_bytes.resize(cfg->nranks);
  for (uint32_t r = 0; r < cfg->nranks; ++r)
    f->heap_bytes[r] = f->ctrl->ranks[r].heap_bytes;
  // ---------------- peer mappings (NVLink P2P inside the process, IPC across)
  std::map<std::pair<int, uint32_t>, char*> opened;  // (device, rank) -> ptr
  f->base.assign(cfg->nlocal, std::vector<char*>(cfg->nranks, nullptr));
  for (uint32_t i = 0; i < cfg->nlocal; ++i) {
    Local* L = f->locals[i].get();
    if (L->device < 0) continue;
    RDMM_CUDA_TRY(cudaSetDevice(L->device));
    for (uint32_t r = 0; r < cfg->nranks; ++r) {
      if (f->ctrl->ranks[r].device < 0) continue;
      if (Local* R = f->local(r)) {
        if (R->device != L->device) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, L->device, R->device);
          if (can) {
            cudaError_t e = cudaDeviceEnablePeerAccess(R->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
              return fail(RDMM_ERR_CUDA, "cudaDeviceEnablePeerAccess failed");
            cudaGetLastError();
          }
        }
        f->base[i][r] = R->heap.base;
      } else {
        auto key = std::make_pair(L->device, r);
        auto it = opened.find(key);
        if (it == opened.end()) {
          void* p = nullptr;
          RDMM_CUDA_TRY(cudaIpcOpenMemHandle(&p, f->ctrl->ranks[r].heap,
                                             cudaIpcMemLazyEnablePeerAccess));
          f->ipc_opened.push_back({L->device, p});
          it = opened.emplace(key, static_cast<char*>(p)).first;
        }
        f->base[i][r] = it->second;
      }
    }
  }
  // every local rank arrives once; after the barrier every rank of every
  // process has mapped every heap, so the shm name is no longer needed
  if (int rc = barrier_n(f.get(), cfg->nlocal)) return rc;
  if (f->shared && f->owns_shm) {
    shm_unlink(f->session.c_str());
    f->owns_shm = false;
  }
  *out = f.release();
  return RDMM_OK;
}

extern "C" void rdmm_fabric_destroy(rdmm_fabric* f) {
  if (!f) return;
  for (auto& [dev, p] : f->ipc_opened) {
    cudaSetDevice(dev);
    cudaIpcCloseMemHandle(p);
  }
  for (auto& L : f->locals) {
    if (L->device < 0) continue;
    cudaSetDevice(L->device);
    for (auto s : L->streams)
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    if (L->atomic_stream) cudaStreamDestroy(L->atomic_stream);
    if (L->heap.base) cudaFree(L->heap.base);
    if (L->atomic_slot) cudaFreeHost(L->atomic_slot);
  }
  bool any_gpu = false;
  for (auto& L : f->locals) any_gpu |= L->device >= 0;
  if (f->ctrl && any_gpu) {
    cudaHostUnregister(f->ctrl);
    cudaGetLastError();
  }
  if (f->ctrl) {
    munmap(f->ctrl, f->ctrl_map_bytes);
  }
  if (f->shared && f->owns_shm) shm_unlink(f->session.c_str());
  delete f;
}

extern "C" uint32_t rdmm_fabric_nranks(const rdmm_fabric* f) { return f->cfg.nranks; }
extern "C" uint32_t rdmm_fabric_node_group(const rdmm_fabric* f) {
  return f->cfg.node_group;
}
extern "C" uint64_t rdmm_fabric_queue_capacity(const rdmm_fabric* f) {
  return f->cfg.queue_capacity;
}
extern "C" int rdmm_fabric_is_local(const rdmm_fabric* f, uint32_t rank) {
  return rank >= f->cfg.first_local && rank < f->cfg.first_local + f->cfg.nlocal;
}
extern "C" int rdmm_fabric_device(const rdmm_fabric* f, uint32_t rank) {
  auto* ff = const_cast<rdmm_fabric*>(f);
  Local* L = ff->local(rank);
  return L ? L->device : -1;
}
extern "C" rdmm_stream_t rdmm_fabric_stream(rdmm_fabric* f, uint32_t rank,
                                            int which) {
  Local* L = f->local(rank);
  if (!L || which < 0 || which > 3) return nullptr;
  return reinterpret_cast<rdmm_stream_t>(L->streams[which]);
}
extern "C" uint64_t rdmm_fabric_next_uid(rdmm_fabric* f) { return ++f->uid; }

extern "C" void rdmm_fabric_abort(rdmm_fabric* f, const char* why) {
  if (!f || !f->ctrl) return;
  uint32_t exp = 0;
  if (f->ctrl->abort.compare_exchange_strong(exp, 1)) {
    std::strncpy(f->ctrl->abort_msg, why ? why : "aborted", sizeof(f->ctrl->abort_msg) - 1);
  }
}

// ------------------------------------------------------------------ heap

extern "C" int rdmm_heap_alloc(rdmm_fabric* f, uint32_t rank, uint64_t nbytes,
                               rdmm_gptr* out) {
  if (rank >= f->cfg.nranks) return fail(RDMM_ERR_FABRIC, "rank out of range");
  Local* L = f->local(rank);
  if (!L)
    return fail(RDMM_ERR_FABRIC,
                "alloc on a rank hosted by another process (owner-only allocation)");
  uint64_t off = 0;
  if (!L->heap.alloc(nbytes, &off)) {
    uint64_t rem = L->heap.remaining;
    return fail(RDMM_ERR_HEAP_EXHAUSTED,
                "shared heap exhausted: requested " + std::to_string(nbytes) +
                    " bytes, " + std::to_string(rem) + " remaining");
  }
  *out = rdmm_gptr{rank, 0, off, nbytes};
  return RDMM_OK;
}

extern "C" int rdmm_heap_free(rdmm_fabric* f, rdmm_gptr p) {
  if (p.rank >= f->cfg.nranks) return fail(RDMM_ERR_FABRIC, "rank out of range");
  Local* L = f->local(p.rank);
  if (!L) return fail(RDMM_ERR_FABRIC, "free on a rank hosted by another process");
  if (!L->heap.release(p.offset))
    return fail(RDMM_ERR_FABRIC, "free of unknown or already-freed allocation");
  return RDMM_OK;
}

extern "C" int rdmm_heap_remaining(const rdmm_fabric* f, uint32_t rank,
                                   uint64_t* out) {
  Local* L = const_cast<rdmm_fabric*>(f)->local(rank);
  if (!L) return fail(RDMM_ERR_FABRIC, "rank not local");
  std::lock_guard<std::mutex> lk(L->heap.mu);
  *out = L->heap.remaining;
  return RDMM_OK;
}

extern "C" int rdmm_gptr_device(rdmm_fabric* f, uint32_t caller, rdmm_gptr p,
                                void** dev) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (int rc = check_gptr(f, p, false)) return rc;
  *dev = dev_addr(f, C, p);
  return RDMM_OK;
}

// ------------------------------------------------------------ transfers

extern "C" int rdmm_get_nb(rdmm_fabric* f, uint32_t caller, rdmm_gptr src,
                           void* dst, rdmm_stream_t stream, rdmm_handle* h) {
  if (h) *h = rdmm_handle{nullptr, 0};
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (int rc = check_gptr(f, src, false)) return rc;
  cudaStream_t s = stream ? as_stream(stream) : C->streams[1];
  RDMM_CUDA_TRY(cudaSetDevice(C->device));
  if (src.length)
    RDMM_CUDA_TRY(cudaMemcpyAsync(dst, dev_addr(f, C, src), src.length,
                                  cudaMemcpyDefault, s));
  f->record_get(src.rank, caller, src.length);
  if (h) {
    cudaEvent_t e;
    RDMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    RDMM_CUDA_TRY(cudaEventRecord(e, s));
    h->event = e;
  }
  return RDMM_OK;
}

extern "C" int rdmm_put_nb(rdmm_fabric* f, uint32_t caller, const void* src,
                           rdmm_gptr dst, rdmm_stream_t stream, rdmm_handle* h) {
  if (h) *h = rdmm_handle{nullptr, 0};
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (int rc = check_gptr(f, dst, false)) return rc;
  cudaStream_t s = stream ? as_stream(stream) : C->streams[1];
  RDMM_CUDA_TRY(cudaSetDevice(C->device));
  if (dst.length)
    RDMM_CUDA_TRY(cudaMemcpyAsync(dev_addr(f, C, dst), src, dst.length,
                                  cudaMemcpyDefault, s));
  f->record_put(caller, dst.rank, dst.length);
  if (h) {
    cudaEvent_t e;
    RDMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    RDMM_CUDA_TRY(cudaEventRecord(e, s));
    h->event = e;
  }
  return RDMM_OK;
}

extern "C" int rdmm_wait(rdmm_fabric* f, rdmm_handle* h, rdmm_stream_t consumer) {
  (void)f;
  if (!h || !h->event) return RDMM_OK;  // idempotent (fabric.hpp:467-471)
  cudaEvent_t e = static_cast<cudaEvent_t>(h->event);
  if (consumer)
    RDMM_CUDA_TRY(cudaStreamWaitEvent(as_stream(consumer), e, 0));
  else
    RDMM_CUDA_TRY(cudaEventSynchronize(e));
  cudaEventDestroy(e);
  h->event = nullptr;
  return RDMM_OK;
}

extern "C" int rdmm_get_host(rdmm_fabric* f, uint32_t caller, rdmm_gptr src,
                             void* dst) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (src.offset & RDMM_CTRL_BIT) {
    if (int rc = check_gptr(f, src, true)) return rc;
    std::memcpy(dst, f->arena + (src.offset & ~RDMM_CTRL_BIT), src.length);
    f->record_get(src.rank, caller, src.length);
    return RDMM_OK;
  }
  if (int rc = check_gptr(f, src, false)) return rc;
  RDMM_CUDA_TRY(cudaSetDevice(C->device));
  if (src.length)
    RDMM_CUDA_TRY(cudaMemcpy(dst, dev_addr(f, C, src), src.length, cudaMemcpyDefault));
  f->record_get(src.rank, caller, src.length);
  return RDMM_OK;
}

extern "C" int rdmm_peek(rdmm_fabric* f, uint32_t caller, rdmm_gptr src,
                         void* dst) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (int rc = check_gptr(f, src, true)) return rc;
  if (src.offset & RDMM_CTRL_BIT) {
    std::memcpy(dst, f->arena + (src.offset & ~RDMM_CTRL_BIT), src.length);
    return RDMM_OK;
  }
  RDMM_CUDA_TRY(cudaSetDevice(C->device));
  if (src.length)
    RDMM_CUDA_TRY(cudaMemcpy(dst, dev_addr(f, C, src), src.length, cudaMemcpyDefault));
  return RDMM_OK;
}

extern "C" int rdmm_put_host(rdmm_fabric* f, uint32_t caller, const void* src,
                             rdmm_gptr dst) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (dst.offset & RDMM_CTRL_BIT) {
    if (int rc = check_gptr(f, dst, true)) return rc;
    std::memcpy(f->arena + (dst.offset & ~RDMM_CTRL_BIT), src, dst.length);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    f->record_put(caller, dst.rank, dst.length);
    return RDMM_OK;
  }
  if (int rc = check_gptr(f, dst, false)) return rc;
  RDMM_CUDA_TRY(cudaSetDevice(C->device));
  if (dst.length)
    RDMM_CUDA_TRY(cudaMemcpy(dev_addr(f, C, dst), src, dst.length, cudaMemcpyDefault));
  f->record_put(caller, dst.rank, dst.length);
  return RDMM_OK;
}

// ------------------------------------------------------------ atomics

extern "C" int rdmm_fetch_add_i64(rdmm_fabric* f, uint32_t caller,
                                  rdmm_gptr cell, int64_t delta, int64_t* old) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (cell.length != 8)
    return fail(RDMM_ERR_FABRIC, "fetch_add: pointer must name one 8-byte integer");
  if ((cell.offset & ~RDMM_CTRL_BIT) % 8 != 0)
    return fail(RDMM_ERR_FABRIC, "fetch_add: misaligned counter");
  if (int rc = check_gptr(f, cell, true)) return rc;
  if (cell.offset & RDMM_CTRL_BIT) {
    auto* p = reinterpret_cast<int64_t*>(f->arena + (cell.offset & ~RDMM_CTRL_BIT));
    *old = __atomic_fetch_add(p, delta, __ATOMIC_SEQ_CST);
  } else {
    // device-heap cell: one system-scope atomic over NVLink from the
    // caller's GPU (slow path; reservations use control cells), on an idle
    // stream so it does not wait for the queued compute
    RDMM_CUDA_TRY(cudaSetDevice(C->device));
    auto* p = reinterpret_cast<unsigned long long*>(dev_addr(f, C, cell));
    k_fetch_add<<<1, 1, 0, C->atomic_stream>>>(p, delta, C->atomic_slot);
    RDMM_CUDA_TRY(cudaStreamSynchronize(C->atomic_stream));
    *old = static_cast<int64_t>(*C->atomic_slot);
  }
  f->record_atomic(caller, cell.rank);
  f->emit(C, 0, caller, cell.rank, 8, 0);
  return RDMM_OK;
}

extern "C" int rdmm_ctrl_cells(rdmm_fabric* f, uint32_t caller, uint64_t tag,
                               uint64_t count, rdmm_gptr* base) {
  if (!f->local(caller)) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  bool fresh = false;
  const uint64_t off = coll_alloc(f, tag, std::max<uint64_t>(count, 1) * 8, &fresh);
  if (off == ~0ull) return fail(RDMM_ERR_HEAP_EXHAUSTED, "control arena exhausted");
  *base = rdmm_gptr{caller, 0, RDMM_CTRL_BIT | off, 8};
  return RDMM_OK;
}

extern "C" int rdmm_ctrl_release(rdmm_fabric* f, uint32_t caller, uint64_t tag) {
  if (!f->local(caller)) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  Ctrl* c = f->ctrl;
  SpinLock lk(c->lock);
  for (uint32_t i = 0; i < c->ncoll; ++i)
    if (c->coll[i].live && c->coll[i].tag == tag) {
      if (++c->coll[i].releases >= c->nranks) c->coll[i].live = 0;
      break;
    }
  while (c->ncoll > 0 && !c->coll[c->ncoll - 1].live) {
    c->arena_used = c->coll[c->ncoll - 1].offset;
    --c->ncoll;
  }
  return RDMM_OK;
}

// ------------------------------------------------------------ queues

namespace {
QueueHdr* queue_at(rdmm_fabric* f, uint64_t qid) {
  return reinterpret_cast<QueueHdr*>(f->arena + qid);
}
QueueSlot* queue_slots(QueueHdr* q) {
  return reinterpret_cast<QueueSlot*>(reinterpret_cast<char*>(q) + sizeof(QueueHdr));
}
}  // namespace

extern "C" int rdmm_queue_open(rdmm_fabric* f, uint32_t caller, uint64_t tag,
                               uint64_t capacity, uint64_t* qids) {
  if (!f->local(caller)) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (capacity == 0) capacity = f->cfg.queue_capacity;
  const uint64_t per = sizeof(QueueHdr) + capacity * sizeof(QueueSlot);
  bool fresh = false;
  const uint64_t off = coll_alloc(f, tag, per * f->cfg.nranks, &fresh);
  if (off == ~0ull) return fail(RDMM_ERR_HEAP_EXHAUSTED, "control arena exhausted by queues");
  for (uint32_t r = 0; r < f->cfg.nranks; ++r) {
    qids[r] = off + r * per;
    if (fresh) {
      QueueHdr* q = queue_at(f, qids[r]);
      q->capacity = capacity;
      q->owner = r;
    }
  }
  // make the zeroed queue headers visible to every rank before first use
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return RDMM_OK;
}

// fabric.hpp:502-514
extern "C" int rdmm_queue_push(rdmm_fabric* f, uint32_t caller, uint64_t qid,
                               rdmm_gptr v, const void* inl, uint32_t inl_bytes) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (inl_bytes > kInline) return fail(RDMM_ERR_INVALID, "queue inline payload > 40 bytes");
  QueueHdr* q = queue_at(f, qid);
  const int64_t t = q->tail.fetch_add(1, std::memory_order_seq_cst);
  if (t - q->head.load(std::memory_order_acquire) >= int64_t(q->capacity))
    return fail(RDMM_ERR_QUEUE_FULL,
                "remote queue full (capacity " + std::to_string(q->capacity) + ")");
  QueueSlot& slot = queue_slots(q)[uint64_t(t) % q->capacity];
  // a slot reused after wrap-around must have been drained
  while (slot.ready.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  slot.v = v;
  slot.inl_bytes = inl_bytes;
  if (inl_bytes) std::memcpy(slot.inl, inl, inl_bytes);
  slot.ready.store(1, std::memory_order_release);
  f->record_atomic(caller, q->owner);
  f->record_put(caller, q->owner, sizeof(rdmm_gptr));
  f->emit(C, 2, caller, q->owner, sizeof(rdmm_gptr), 0);
  return RDMM_OK;
}

// fabric.hpp:517-528
extern "C" int rdmm_queue_pop(rdmm_fabric* f, uint32_t caller, uint64_t qid,
                              rdmm_gptr* v, void* inl, uint32_t inl_bytes,
                              int* got) {
  *got = 0;
  if (!f->local(caller)) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  QueueHdr* q = queue_at(f, qid);
  if (q->owner != caller)
    return fail(RDMM_ERR_FABRIC, "queue_pop: caller is not the queue owner");
  const int64_t h = q->head.load(std::memory_order_relaxed);
  QueueSlot& slot = queue_slots(q)[uint64_t(h) % q->capacity];
  if (slot.ready.load(std::memory_order_acquire) == 0) return RDMM_OK;
  *v = slot.v;
  if (inl && inl_bytes) std::memcpy(inl, slot.inl, std::min(inl_bytes, kInline));
  slot.ready.store(0, std::memory_order_release);
  q->head.store(h + 1, std::memory_order_release);
  *got = 1;
  return RDMM_OK;
}

// ------------------------------------------------------------ barrier

extern "C" int rdmm_barrier(rdmm_fabric* f, uint32_t caller) {
  Local* C = f->local(caller);
  if (!C) return fail(RDMM_ERR_FABRIC, "caller rank not local");
  if (C->device >= 0) {
    cudaSetDevice(C->device);
    for (auto s : C->streams) RDMM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  return barrier_n(f, 1);
}

// ------------------------------------------------------------ traffic log

extern "C" void rdmm_set_phase(rdmm_fabric* f, uint32_t caller, int64_t label) {
  if (Local* L = f->local(caller)) L->label = label;
}
extern "C" int64_t rdmm_phase(rdmm_fabric* f, uint32_t caller) {
  Local* L = f->local(caller);
  return L ? L->label : 0;
}
extern "C" void rdmm_record_tile_fetch(rdmm_fabric* f, uint32_t caller,
                                       uint32_t owner, int matrix, uint32_t i,
                                       uint32_t j) {
  Local* L = f->local(caller);
  std::lock_guard<std::mutex> lk(f->tmu);
  f->fetches.push_back({owner, caller, L ? L->label : 0, matrix, i, j});
}
extern "C" void rdmm_emit_compute(rdmm_fabric* f, uint32_t caller, uint64_t flops) {
  f->emit(f->local(caller), 1, caller, caller, 0, flops);
}
extern "C" void rdmm_record_self_get(rdmm_fabric* f, uint32_t caller, uint64_t bytes) {
  f->record_get(caller, caller, bytes);
}
extern "C" void rdmm_record_get(rdmm_fabric* f, uint32_t caller, uint32_t owner,
                                uint64_t bytes) {
  f->record_get(owner, caller, bytes);
}
extern "C" int rdmm_traffic_pair(const rdmm_fabric* f, uint32_t src, uint32_t dst,
                                 rdmm_traffic* out) {
  std::lock_guard<std::mutex> lk(f->tmu);
  *out = rdmm_traffic{};
  for (const auto& [k, c] : f->cells)
    if (std::get<0>(k) == src && std::get<1>(k) == dst) {
      out->bytes_put += c.bytes_put;
      out->bytes_got += c.bytes_got;
      out->puts += c.puts;
      out->gets += c.gets;
      out->atomic_ops += c.atomic_ops;
    }
  return RDMM_OK;
}
extern "C" int rdmm_traffic_total(const rdmm_fabric* f, rdmm_traffic* out) {
  std::lock_guard<std::mutex> lk(f->tmu);
  *out = rdmm_traffic{};
  for (const auto& [k, c] : f->cells) {
    out->bytes_put += c.bytes_put;
    out->bytes_got += c.bytes_got;
    out->puts += c.puts;
    out->gets += c.gets;
    out->atomic_ops += c.atomic_ops;
  }
  return RDMM_OK;
}
extern "C" void rdmm_traffic_clear(rdmm_fabric* f) {
  std::lock_guard<std::mutex> lk(f->tmu);
  f->cells.clear();
  f->fetches.clear();
}
extern "C" uint64_t rdmm_tile_fetches(const rdmm_fabric* f, rdmm_tile_fetch* out,
                                      uint64_t cap) {
  std::lock_guard<std::mutex> lk(f->tmu);
  const uint64_t n = f->fetches.size();
  for (uint64_t i = 0; i < n && i < cap; ++i) out[i] = f->fetches[i];
  return n;
}
extern "C" void rdmm_event_sink(rdmm_fabric* f, uint32_t caller, int enable) {
  if (Local* L = f->local(caller)) {
    L->sink = enable != 0;
    L->events.clear();
  }
}
extern "C" uint64_t rdmm_events(const rdmm_fabric* f, uint32_t rank,
                                rdmm_event* out, uint64_t cap) {
  Local* L = const_cast<rdmm_fabric*>(f)->local(rank);
  if (!L) return 0;
  const uint64_t n = L->events.size();
  for (uint64_t i = 0; i < n && i < cap; ++i) out[i] = L->events[i];
  return n;
}

// ------------------------------------------------------------ device helpers

extern "C" int rdmm_dev_alloc(rdmm_fabric* f, uint32_t rank, uint64_t bytes,
                              rdmm_stream_t stream, void** out) {
  Local* L = f ? f->local(rank) : nullptr;
  if (L) RDMM_CUDA_TRY(cudaSetDevice(L->device));
  cudaStream_t s = stream ? as_stream(stream) : (L ? L->streams[0] : nullptr);
  RDMM_CUDA_TRY(cudaMallocAsync(out, bytes ? bytes : 16, s));
  return RDMM_OK;
}
extern "C" int rdmm_dev_free(rdmm_fabric* f, uint32_t rank, void* p,
                             rdmm_stream_t stream) {
  if (!p) return RDMM_OK;
  Local* L = f ? f->local(rank) : nullptr;
  if (L) RDMM_CUDA_TRY(cudaSetDevice(L->device));
  cudaStream_t s = stream ? as_stream(stream) : (L ? L->streams[0] : nullptr);
  RDMM_CUDA_TRY(cudaFreeAsync(p, s));
  return RDMM_OK;
}
extern "C" int rdmm_memcpy(void* dst, const void* src, uint64_t bytes,
                           rdmm_stream_t stream) {
  if (!bytes) return RDMM_OK;
  if (stream)
    RDMM_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  else
    RDMM_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  return RDMM_OK;
}
extern "C" int rdmm_memset(void* dst, int value, uint64_t bytes,
                           rdmm_stream_t stream) {
  if (!bytes) return RDMM_OK;
  if (stream)
    RDMM_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, as_stream(stream)));
  else
    RDMM_CUDA_TRY(cudaMemset(dst, value, bytes));
  return RDMM_OK;
}
extern "C" int rdmm_event_record(rdmm_stream_t stream, void** event) {
  cudaEvent_t e;
  RDMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  RDMM_CUDA_TRY(cudaEventRecord(e, as_stream(stream)));
  *event = e;
  return RDMM_OK;
}
extern "C" int rdmm_timing_event_record(rdmm_stream_t stream, void** event) {
  cudaEvent_t e;
  RDMM_CUDA_TRY(cudaEventCreate(&e));
  RDMM_CUDA_TRY(cudaEventRecord(e, as_stream(stream)));
  *event = e;
  return RDMM_OK;
}
extern "C" int rdmm_event_elapsed_ms(void* a, void* b, float* ms) {
  RDMM_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(b)));
  RDMM_CUDA_TRY(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
  return RDMM_OK;
}
extern "C" int rdmm_event_query(void* event, int* done) {
  cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  if (e == cudaSuccess) {
    *done = 1;
    return RDMM_OK;
  }
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    *done = 0;
    return RDMM_OK;
  }
  return fail(RDMM_ERR_CUDA, std::string("event query: ") + cudaGetErrorString(e));
}
extern "C" int rdmm_event_wait(void* event, rdmm_stream_t consumer) {
  RDMM_CUDA_TRY(cudaStreamWaitEvent(as_stream(consumer), static_cast<cudaEvent_t>(event), 0));
  return RDMM_OK;
}
extern "C" int rdmm_event_sync(void* event) {
  RDMM_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(event)));
  return RDMM_OK;
}
extern "C" void rdmm_event_destroy(void* event) {
  if (event) cudaEventDestroy(static_cast<cudaEvent_t>(event));
}
extern "C" int rdmm_stream_sync(rdmm_stream_t stream) {
  RDMM_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  return RDMM_OK;
}
extern "C" int rdmm_get_device(int* device) {
  RDMM_CUDA_TRY(cudaGetDevice(device));
  return RDMM_OK;
}
extern "C" int rdmm_set_device(int device) {
  RDMM_CUDA_TRY(cudaSetDevice(device));
  return RDMM_OK;
}

extern "C" int rdmm_device_count(int* n) {
  RDMM_CUDA_TRY(cudaGetDeviceCount(n));
  return RDMM_OK;
}

extern "C" int rdmm_memcpy2d(void* dst, uint64_t dpitch, const void* src,
                             uint64_t spitch, uint64_t width_bytes,
                             uint64_t rows, rdmm_stream_t stream) {
  if (!rows || !width_bytes) return RDMM_OK;
  if (stream)
    RDMM_CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, rows,
                                    cudaMemcpyDefault, as_stream(stream)));
  else
    RDMM_CUDA_TRY(cudaMemcpy2D(dst, dpitch, src, spitch, width_bytes, rows,
                               cudaMemcpyDefault));
  return RDMM_OK;
}

extern "C" void* rdmm_ctrl_host(rdmm_fabric* f, rdmm_gptr p) {
  if (!(p.offset & RDMM_CTRL_BIT)) return nullptr;
  return f->arena + (p.offset & ~RDMM_CTRL_BIT);
}
