// common.cu -- error plumbing and per-thread scratch for the C-ABI.
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace rdmm_impl {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

namespace {
struct ScratchKey {
  int dev;
  cudaStream_t stream;
  int slot;
  bool operator<(const ScratchKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    if (stream != o.stream) return stream < o.stream;
    return slot < o.slot;
  }
};
struct ScratchBuf {
  void* p = nullptr;
  size_t n = 0;
};
std::mutex g_scratch_mu;
std::map<ScratchKey, ScratchBuf>& scratch_map() {
  static auto* m = new std::map<ScratchKey, ScratchBuf>();  // never destroyed
  return *m;
}
}  // namespace

void* scratch(size_t bytes, int slot, cudaStream_t stream) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  ScratchBuf& b = scratch_map()[ScratchKey{dev, stream, slot}];
  if (b.n >= bytes && b.p) return b.p;
  if (b.p) cudaFreeAsync(b.p, stream);
  b.p = nullptr;
  b.n = 0;
  const size_t n = bytes + bytes / 4 + 4096;
  if (cudaMallocAsync(&b.p, n, stream) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return nullptr;
  }
  b.n = n;
  return b.p;
}

static std::atomic<unsigned long long> g_launches{0};
void count_launch(unsigned n) { g_launches += n; }

namespace {
struct TimingState {
  std::mutex mu;
  bool on = false;
  struct Rec {
    cudaEvent_t a, b;
    int kind;
  };
  std::vector<Rec> recs;
};
TimingState& timing() {
  static TimingState t;
  return t;
}
}  // namespace

KernelTimer::KernelTimer(cudaStream_t s, int k) : stream(s), kind(k) {
  auto& t = timing();
  if (!t.on) return;
  cudaEventCreate(&start);
  cudaEventRecord(start, s);
}
KernelTimer::~KernelTimer() {
  if (!start) return;
  cudaEvent_t end;
  cudaEventCreate(&end);
  cudaEventRecord(end, stream);
  auto& t = timing();
  std::lock_guard<std::mutex> lk(t.mu);
  t.recs.push_back({start, end, kind});
}

}  // namespace rdmm_impl

extern "C" unsigned long long rdmm_kernel_launches(void) {
  return rdmm_impl::g_launches.load();
}

extern "C" void rdmm_kernel_timing(int enable) {
  auto& t = rdmm_impl::timing();
  std::lock_guard<std::mutex> lk(t.mu);
  t.on = enable != 0;
  for (auto& r : t.recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  t.recs.clear();
}

extern "C" int rdmm_kernel_timing_get(int kind, double* total_ms,
                                      unsigned long long* count) {
  auto& t = rdmm_impl::timing();
  std::lock_guard<std::mutex> lk(t.mu);
  double ms = 0;
  unsigned long long n = 0;
  for (auto& r : t.recs) {
    if (kind >= 0 && r.kind != kind) continue;
    cudaEventSynchronize(r.b);
    float x = 0;
    cudaEventElapsedTime(&x, r.a, r.b);
    ms += x;
    ++n;
  }
  *total_ms = ms;
  *count = n;
  return 0;
}

extern "C" int rdmm_impl_fail(int code, const char* msg) {
  return rdmm_impl::fail(code, msg ? msg : "");
}

extern "C" const char* rdmm_last_error(void) {
  return rdmm_impl::g_last_error.c_str();
}

extern "C" const char* rdmm_version(void) {
  return "rdmm-b200 0.1 (sm_100a)";
}
