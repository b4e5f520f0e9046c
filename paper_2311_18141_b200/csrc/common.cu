// common.cu -- error plumbing and per-thread scratch for the C-ABI.
#include <atomic>
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
struct Scratch {
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
  };
  // [device][slot]
  std::vector<std::vector<Buf>> bufs;
  ~Scratch() {
    // Process teardown: the CUDA context may already be gone; leak quietly.
  }
};
thread_local Scratch g_scratch;
}  // namespace

void* scratch(size_t bytes, int slot) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto& per = g_scratch.bufs;
  if (per.size() <= size_t(dev)) per.resize(dev + 1);
  auto& slots = per[dev];
  if (slots.size() <= size_t(slot)) slots.resize(slot + 1);
  auto& b = slots[slot];
  if (b.n >= bytes) return b.p;
  if (b.p) {
    cudaDeviceSynchronize();  // in-flight kernels may still use the old one
    cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
  }
  size_t n = bytes + bytes / 4 + 4096;
  if (cudaMalloc(&b.p, n) != cudaSuccess) {
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
