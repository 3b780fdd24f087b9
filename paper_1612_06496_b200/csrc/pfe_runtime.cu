// Host runtime + C ABI of the B200 PFE solver (include/pfe_b200.h).
//
// Owns device memory, the operator set-up (sparse.cpp:96-122, pcg.cpp:9-29
// restated for the device layouts), and the drivers of the nested Bregman
// loop (solver.cpp:73-136).  The PCG loop runs either host-driven (one
// control-block read per PCG iteration; needed for callbacks and the
// relative-change stopping test) or as a CUDA graph whose PCG loop is a
// device-side conditional WHILE node, so a whole soc / two_stage run is one
// graph launch with no host round trips.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "pfe_b200.h"
#include "pfe_errors.h"
#include "pfe_kernels.cuh"
#include "pfe_launch.h"
#include "pfe_polar.cuh"

using pfe_dev::Ctl;
using pfe_dev::PcgArgs;
using pfe_dev::SbArgs;
using pfe_host::Error;
using pfe_host::LaunchTable;
using pfe_host::TopoDesc;

namespace {

thread_local std::string g_last_error;
constexpr int kTraceCap = 1 << 16;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw Error(PFE_CUDA_ERROR, std::string(#x) + " failed: " + cudaGetErrorString(e_));      \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PFE_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return PFE_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PFE_CUDA_ERROR;
  }
}

[[noreturn]] void config_error(const std::string& m) { throw Error(PFE_CONFIG_ERROR, m); }

void require_device(int dev) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    config_error("no CUDA device available: the B200 PFE solver has no CPU fallback");
  if (dev < 0 || dev >= count) config_error("CUDA device ordinal out of range");
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) {
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, dev));
    config_error(std::string("device ") + prop.name + " is not sm_100-class; this library is built for sm_100a only");
  }
  CK(cudaSetDevice(dev));
}

// Owner of a set of device allocations.  Allocations are stream-ordered
// (cudaMallocAsync / cudaFreeAsync on the owner's stream) from the device's
// default memory pool, which keeps freed memory (release threshold: never),
// so creating and destroying solvers and states in a loop -- the one-call
// C ABI does that on every call -- re-uses device memory instead of paying
// cudaMalloc / cudaFree each time.
void retain_pool_memory(int dev) {
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = ~static_cast<uint64_t>(0);
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done[dev] = true;
}

// NVTX range for a scope (the reference has no tracer; profilers
// see the stages of a call as named ranges: `ncu --nvtx --nvtx-include "pfe projection/"`).
// NVTX 3 is header-only and does nothing unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Process-wide pool of host worker threads for parallel_for: creating 16
// std::threads per call cost ~0.5 ms, which made the many small parallel
// loops of the general-graph set-up (one per breadth-first level) slower
// than serial.  Workers sleep on a condition variable between jobs; one job
// runs at a time (callers from several host threads queue on `run_mu`); a
// parallel_for issued from inside a worker runs inline.
struct HostPool {
  std::mutex run_mu;  // one job at a time
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::vector<std::thread> workers;
  const std::function<void(long, long)>* job = nullptr;
  long n = 0, per = 0;
  int parts = 0, next_part = 0, pending = 0;
  unsigned long gen = 0;
  bool stop = false;
  static thread_local bool in_worker;

  explicit HostPool(int nthreads) {
    for (int w = 0; w < nthreads; ++w) workers.emplace_back([this] { loop(); });
  }
  // run part p of the current job (mu not held)
  void run_part(int p) {
    const long b = p * per, e = std::min(n, b + per);
    if (b < e) (*job)(b, e);
  }
  void loop() {
    in_worker = true;
    unsigned long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return stop || (gen != seen && next_part < parts); });
      if (stop) return;
      while (next_part < parts) {
        const int p = next_part++;
        lk.unlock();
        run_part(p);
        lk.lock();
        if (--pending == 0) done_cv.notify_all();
      }
      seen = gen;
    }
  }
  void run(long total, int t, const std::function<void(long, long)>& f) {
    std::lock_guard<std::mutex> serial(run_mu);
    std::unique_lock<std::mutex> lk(mu);
    job = &f;
    n = total;
    parts = t;
    per = (total + t - 1) / t;
    next_part = 0;
    pending = t;
    ++gen;
    cv.notify_all();
    in_worker = true;  // a parallel_for inside f on this thread runs inline
    while (next_part < parts) {  // the caller works too
      const int p = next_part++;
      lk.unlock();
      run_part(p);
      lk.lock();
      --pending;
    }
    in_worker = false;
    done_cv.wait(lk, [&] { return pending == 0; });
    job = nullptr;
  }
};
thread_local bool HostPool::in_worker = false;

HostPool& host_pool() {
  // never destroyed: workers live for the process.  A forked child has no
  // copies of the parent's threads, so it builds its own pool.
  static std::mutex mu;
  static HostPool* pool = nullptr;
  static pid_t owner = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (!pool || owner != getpid()) {
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    pool = new HostPool(std::min(hw, 16) - 1);
    owner = getpid();
  }
  return *pool;
}

// f(begin, end) over [0, n) on up to 16 host threads (chunks of >= grain
// items; small inputs run inline).  f must not throw.
template <class F>
void parallel_for(long n, F&& f, long grain = 1L << 16) {
  const long hw = std::max(1u, std::thread::hardware_concurrency());
  const int t = static_cast<int>(std::min<long>(std::min<long>(hw, 16), (n + grain - 1) / std::max(1L, grain)));
  if (t <= 1 || HostPool::in_worker) {
    f(0L, n);
    return;
  }
  const std::function<void(long, long)> fn = [&f](long b, long e) { f(b, e); };
  host_pool().run(n, t, fn);
}

// Large copies between pageable host memory and the device go through two
// process-wide 32 MB pinned bounce buffers, the host side of each chunk
// copied by several threads (a pageable cudaMemcpy ran at ~2 GB/s, e.g.
// 0.5 s to download C4's 1 GB embedding).
struct PinnedStage {
  std::mutex mu;
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  static constexpr size_t kCap = 32u << 20;
  bool ok = false;
  std::once_flag once;
  bool ready() {  // thread-safe lazy set-up (several solvers may share a device)
    std::call_once(once, [this] {
      ok = cudaMallocHost(&buf[0], kCap) == cudaSuccess && cudaMallocHost(&buf[1], kCap) == cudaSuccess &&
           cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) == cudaSuccess;
      if (!ok) cudaGetLastError();
    });
    return ok;
  }
};
// One stage per device: its events belong to that device's streams (a
// multi-GPU solve drives several devices from one process).
PinnedStage& pinned_stage() {
  static PinnedStage* stages = new PinnedStage[64];  // never destroyed: no CUDA calls at exit
  int dev = 0;
  cudaGetDevice(&dev);
  return stages[dev >= 0 && dev < 64 ? dev : 0];
}
void par_memcpy(void* dst, const void* src, size_t bytes) {
  parallel_for(static_cast<long>(bytes), [&](long b, long e) {
    std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, static_cast<size_t>(e - b));
  }, 1L << 21);
}
constexpr size_t kStageMin = 16u << 20;  // smaller copies go direct

// Page-locked (cudaMallocHost / cudaHostRegister) host memory: the DMA
// engine reads it directly, no bounce buffer needed.
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: a plain pageable pointer is not an error
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  PinnedStage& ps = pinned_stage();
  if (bytes < kStageMin || host_pinned(src) || !ps.ready()) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  std::lock_guard<std::mutex> lk(ps.mu);
  int i = 0;
  for (size_t off = 0; off < bytes; off += PinnedStage::kCap, i ^= 1) {
    const size_t n = std::min(PinnedStage::kCap, bytes - off);
    CK(cudaEventSynchronize(ps.ev[i]));  // the previous copy out of this buffer is done
    par_memcpy(ps.buf[i], static_cast<const char*>(src) + off, n);
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, ps.buf[i], n, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(ps.ev[i], s));
  }
}

// Blocking: returns when dst holds the data.
void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  PinnedStage& ps = pinned_stage();
  if (bytes < kStageMin || host_pinned(dst) || !ps.ready()) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  std::lock_guard<std::mutex> lk(ps.mu);
  const size_t cap = PinnedStage::kCap;
  const size_t nchunks = (bytes + cap - 1) / cap;
  auto issue = [&](size_t c) {
    const size_t off = c * cap, n = std::min(cap, bytes - off);
    // an earlier copy_h2d (another solver's stream) may still be reading this buffer
    CK(cudaStreamWaitEvent(s, ps.ev[c & 1], 0));
    CK(cudaMemcpyAsync(ps.buf[c & 1], static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ps.ev[c & 1], s));
  };
  issue(0);
  if (nchunks > 1) issue(1);
  for (size_t c = 0; c < nchunks; ++c) {
    CK(cudaEventSynchronize(ps.ev[c & 1]));
    const size_t off = c * cap, n = std::min(cap, bytes - off);
    par_memcpy(static_cast<char*>(dst) + off, ps.buf[c & 1], n);
    if (c + 2 < nchunks) issue(c + 2);
  }
}

// Copy on a (non-blocking) solver stream and wait: ordered after that
// stream's kernels, which a legacy-stream cudaMemcpy is not.
void stream_copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
  CK(cudaStreamSynchronize(s));
}

// Makes `dev` current for a scope and restores the caller's device after
// (destroy entry points free memory and graphs that belong to `dev`).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Process-wide pool of pinned host control blocks: cudaMallocHost /
// cudaFreeHost cost milliseconds each (cudaFreeHost synchronizes the
// device), which showed up as ~7 ms per pfe_solve call on small graphs.
struct PinnedCtlPool {
  std::mutex mu;
  std::vector<void*> free_list;
  void* get(size_t bytes) {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (!free_list.empty()) {
        void* p = free_list.back();
        free_list.pop_back();
        return p;
      }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
  }
  void put(void* p) {
    std::lock_guard<std::mutex> lk(mu);
    free_list.push_back(p);
  }
};
PinnedCtlPool& pinned_ctl_pool() {
  static PinnedCtlPool* pool = new PinnedCtlPool();  // never destroyed: no CUDA calls at exit
  return *pool;
}

// std::vector whose elements are left uninitialised on resize (PODs that
// are written before they are read): big set-up buffers are then not
// zero-filled serially before the parallel loops fill them.
template <class T>
struct UninitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <class U>
  UninitAlloc(const UninitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using uvec = std::vector<T, UninitAlloc<T>>;

// Exact-size cache of large device blocks in front of cudaMallocAsync.  The
// one-call C ABI (pfe_solve) builds and destroys a solver and a state per
// call; for C4 that is 13 state arrays of 1-4.3 GB.  The driver's pool does
// keep freed memory, but re-carving it for the next call cost 140-1400 ms per
// call (measured under bench.py, gpurun_out/bench_e2e_c4.err), several times
// the copies themselves.  Blocks >= kMin bytes released at destruction --
// when nothing is pending on them: every entry point synchronises its stream
// before it returns -- are parked here per device and handed back to the next
// allocation of exactly that size.  The cache holds at most `cap` bytes per
// device (PFE_CACHE_MB, default 40 % of device memory; 0 disables it); on an
// allocation failure it is flushed and the allocation retried.
struct BlockCache {
  static constexpr size_t kMin = 8u << 20;
  struct PerDev {
    std::multimap<size_t, void*> blocks;
    size_t bytes = 0;
    size_t cap = 0;
    bool cap_set = false;
  };
  std::mutex mu;
  PerDev dev[64];
  static int current() {
    int d = 0;
    cudaGetDevice(&d);
    return d >= 0 && d < 64 ? d : 0;
  }
  void set_cap(PerDev& pd) {
    if (pd.cap_set) return;
    pd.cap_set = true;
    if (const char* e = std::getenv("PFE_CACHE_MB")) {
      pd.cap = static_cast<size_t>(std::strtoull(e, nullptr, 10)) << 20;
      return;
    }
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      tot = 0;
    }
    pd.cap = tot / 5 * 2;
  }
  void* take(size_t bytes) {
    if (bytes < kMin) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    PerDev& pd = dev[current()];
    auto it = pd.blocks.find(bytes);
    if (it == pd.blocks.end()) return nullptr;
    void* p = it->second;
    pd.blocks.erase(it);
    pd.bytes -= bytes;
    return p;
  }
  bool park(void* p, size_t bytes) {
    if (bytes < kMin) return false;
    std::lock_guard<std::mutex> lk(mu);
    PerDev& pd = dev[current()];
    set_cap(pd);
    if (pd.bytes + bytes > pd.cap) return false;
    pd.blocks.emplace(bytes, p);
    pd.bytes += bytes;
    return true;
  }
  // returns the cached bytes it gave back to the driver's pool
  size_t flush() {
    std::lock_guard<std::mutex> lk(mu);
    PerDev& pd = dev[current()];
    const size_t was = pd.bytes;
    for (auto& kv : pd.blocks) cudaFreeAsync(kv.second, nullptr);
    pd.blocks.clear();
    pd.bytes = 0;
    if (was) cudaStreamSynchronize(nullptr);
    return was;
  }
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();  // never destroyed: no CUDA calls at exit
  return *c;
}

struct DevPool {
  struct Block {
    void* p;
    size_t bytes;
  };
  std::vector<Block> ptrs;
  cudaStream_t stream = nullptr;   // allocation stream, set before the first allocation
  cudaStream_t fstream = nullptr;  // free stream: a state may outlive its solver's
                                   // stream, so states free on the legacy stream (every
                                   // call synchronizes before returning: nothing pending)
  template <class T>
  T* alloc(size_t count) {
    if (count == 0) count = 1;
    const size_t bytes = count * sizeof(T);
    void* p = block_cache().take(bytes);
    if (!p) {
      cudaError_t e = cudaMallocAsync(&p, bytes, stream);
      if (e == cudaErrorMemoryAllocation && block_cache().flush() > 0) {
        cudaGetLastError();
        e = cudaMallocAsync(&p, bytes, stream);
      }
      CK(e);
    }
    ptrs.push_back({p, bytes});
    return static_cast<T*>(p);
  }
  template <class T, class A>
  T* upload(const std::vector<T, A>& v, cudaStream_t s) {
    T* d = alloc<T>(v.size());
    if (!v.empty()) copy_h2d(d, v.data(), v.size() * sizeof(T), s);
    return d;
  }
  // mid-lifetime release: stream-ordered (work on the block may be pending)
  void release(void* p) {
    auto it = std::find_if(ptrs.begin(), ptrs.end(), [p](const Block& b) { return b.p == p; });
    if (it != ptrs.end()) {
      cudaFreeAsync(p, fstream);
      ptrs.erase(it);
    }
  }
  // at destruction: nothing is pending on the blocks (see BlockCache)
  void free_all() {
    // parked blocks go to the next owner on any stream: make sure the device
    // is done with them (idle in the normal case; an exception unwinding a
    // call may leave work queued)
    for (const Block& b : ptrs)
      if (b.bytes >= BlockCache::kMin) {
        cudaDeviceSynchronize();
        break;
      }
    for (const Block& b : ptrs)
      if (!block_cache().park(b.p, b.bytes)) cudaFreeAsync(b.p, fstream);
    ptrs.clear();
  }
  ~DevPool() { free_all(); }
};

// Per-kernel-class CUDA-event timing (pfe_exec.profile).
struct Prof {
  bool on = false;
  struct Pair {
    cudaEvent_t a, b;
    int cls;
  };
  std::vector<Pair> pool;
  size_t used = 0;
  double ms[PFE_KERNEL_CLASSES] = {};
  int64_t cnt[PFE_KERNEL_CLASSES] = {};
  int cur = -1;
  void begin(int cls, cudaStream_t s) {
    if (!on) return;
    if (used == pool.size()) {
      Pair p{};
      CK(cudaEventCreate(&p.a));
      CK(cudaEventCreate(&p.b));
      pool.push_back(p);
    }
    pool[used].cls = cls;
    CK(cudaEventRecord(pool[used].a, s));
    cur = static_cast<int>(used);
  }
  void end(cudaStream_t s) {
    if (!on) return;
    CK(cudaEventRecord(pool[cur].b, s));
    ++used;
    if (used >= 4096) collect();
  }
  void collect() {
    if (!on || used == 0) return;
    CK(cudaEventSynchronize(pool[used - 1].b));
    for (size_t i = 0; i < used; ++i) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, pool[i].a, pool[i].b));
      ms[pool[i].cls] += t;
      cnt[pool[i].cls] += 1;
    }
    used = 0;
  }
  ~Prof() {
    for (auto& p : pool) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
  }
};

// Host bookkeeping of a state that a captured call advances.
struct Book {
  double* y;
  double* y2;
  int eb_cur;
  bool inner_zero;
  bool rq_valid;
};

struct GraphEntry {
  cudaGraphExec_t exec;
  Book post;    // bookkeeping after the call
  long inner;   // inner iterations the call runs
};

struct GraphCache {
  std::map<std::tuple<int, int, int, int, int, int, int>, GraphEntry> execs;
  ~GraphCache() {
    for (auto& kv : execs) cudaGraphExecDestroy(kv.second.exec);
  }
};

}  // namespace

// ============================================================== solver ====
// Set when NCCL is loaded (row-band solvers own a communicator).
static void (*g_comm_destroy)(void*) = nullptr;

// Device view of an IC(0) factor (see k_ic_apply).
struct IcSweep {
  // rows of one triangular sweep in level order: slot t solves storage row
  // spos[t] with sdg[t] and the slen[t] entries ecol/eval[sbeg[t] ...] in
  // the reference's subtraction order; slots of level l: [lev[l], lev[l+1])
  const int* spos;
  const int* sbeg;
  const int* slen;
  const double* sdg;
  const int* ecol;  // storage position of the operand row
  const double* eval;
  const int* lev;
  int nl;
};
struct IcDev {
  IcSweep fwd, bwd;
};

struct pfe_solver {
  int device = 0;
  cudaStream_t stream = nullptr, aux = nullptr;
  int sm = 148;
  bool use_graphs = true, warn = true;
  bool persistent = true;  // grid topologies: one cooperative launch per split_bregman call
  bool resident = true;    // ... with the PCG state resident in shared memory when it fits
  int persist_kind = 0;    // variant of the last persistent launch (pfe_report::persistent_kind)
  int row_lo = 0, row_hi = -1;  // owned rows of a row-band solver (-1: every row)
  // Row-band (multi-GPU) solver: this solver owns global image rows
  // [band_r0, band_r1) of a band_h x band_w grid and stores local rows
  // [band_lo, band_lo + H_local) (owned rows plus an R-row halo).
  int nranks = 1, rank = 0;
  int band_h = 0, band_w = 0, band_rad = 0, band_r0 = 0, band_r1 = 0, band_lo = 0, band_maxrows = 0;
  long global_n = 0;
  void* comm = nullptr;           // ncclComm_t of this band (one per process, or one per device of a
                                  // single-process multi-GPU team)
  int band_chunk_hint = 4;        // PCG iterations the host issues before reading the control block
  double* tot_local = nullptr;    // [3 d] this band's totals
  double* gathered_a = nullptr;   // [ranks][3 d]
  double* gathered_b = nullptr;   // [ranks][d]
  double* rgather = nullptr;      // [ranks * qr_blocks][d][d] TSQR factors of every band
  double* ystage = nullptr;       // [max owned rows][d] owned-row staging for gathers
  double* yall = nullptr;         // [ranks][max owned rows][d]
  // Multi-GPU partition kind: 0 none, 1 pixel-grid row bands, 2 vertex ranges
  // of a general graph.  Owned rows are [own_vb, own_vb + own_cnt) of the
  // local storage; the others are halo (bands) or ghost (ranges) copies.
  int part = 0;
  long own_vb = 0;
  int own_cnt = 0;
  int max_own = 0;                // largest owned-row count over all ranks
  // Vertex ranges: ghost exchange with every peer rank.
  struct Peer {
    int rank;
    int send_cnt;      // owned rows the peer holds as ghosts (packed in send order)
    int* send_rows;    // device list of those local rows
    long send_off;     // offset (rows) of this peer's block in sendbuf
    int recv_off;      // local row of the first ghost owned by the peer
    int recv_cnt;
  };
  std::vector<Peer> peers;
  double* sendbuf = nullptr;      // [sum send_cnt][d]
  std::vector<int> range_start;   // [ranks + 1] storage-order positions owned by each rank
  std::vector<int> range_vertex;  // storage-order position -> global vertex
  std::vector<int> local_vertex;  // local row (owned, then ghosts) -> global vertex
  unsigned long long* trace = nullptr;  // PFE_TRACE=1: phase trace of the persistent kernel
  pfe_params prm{};
  int n = 0;
  long m = 0;
  int d = 0;
  TopoDesc topo;
  std::vector<long> edge_row;  // edge e -> row of the device edge arrays (host copy)
  int32_t* d_edge_slot = nullptr;  // device copy when the grid topology was built on the device
  // General graphs store vertices in a locality order (BFS): perm_h[v] = the
  // device row of vertex v (empty / null: identity).  Only storage moves; every
  // row keeps its terms in the reference's order.
  std::vector<int> perm_h;
  int* perm_d = nullptr;
  long edge_rows = 0;
  DevPool mem;
  double *deg = nullptr, *sqd = nullptr, *diag = nullptr, *invd = nullptr;
  Ctl* ctl = nullptr;
  Ctl* h_ctl = nullptr;  // pinned mirror
  double* partials = nullptr;    // init / update partials (and objective, norms)
  double* partials_b = nullptr;  // spmv partials
  double* totals = nullptr;      // PCG grid totals written by the producers' last block [4][kMaxD]
  double* partials_c = nullptr;  // init partials of the resident persistent kernel (two sets)
  int max_grid = 0;
  double* rbuf = nullptr;
  int qr_blocks = 1;
  double* wmat = nullptr;
  int* log_it = nullptr;
  int* log_st = nullptr;
  double* log_rel = nullptr;
  long log_cap = 0;
  long inner_launched = 0;  // host mirror of ctl->inner_count
  const LaunchTable* tab = nullptr;
  bool jacobi_fallback = false;
  // IC(0) preconditioner (PFE_PRECOND_IC0 on single-GPU solvers): device
  // factor + level schedules, and the z buffer of the PCG loop
  bool ic = false;
  IcDev icd{};
  double* zbuf = nullptr;
  // Row-band / vertex-range solvers with IC(0): the factor of the GLOBAL
  // matrix lives on every rank (icd), each rank applies it to the gathered
  // global residual (rfull -> zbuf, both [global n][d] in the team's global
  // row order) and uses its own rows of z (pfe_band.cuh: team_pcg).
  bool ic_team = false;
  double* rfull = nullptr;
  double* ic_part = nullptr;  // block partials of the global r.z reduction
  double* ones = nullptr;  // [local n] 1.0: the tiled SpMV forms 1.0 * z + beta p
  double setup_s = 0.0;
  int pred_iters = 1;
  Prof prof;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;  // device time of the last split_bregman / run_soc / two_stage call

  ~pfe_solver() {
    // Large blocks are parked in the block cache for the next solver (any
    // stream): nothing may be pending on them.  Normal calls have already
    // synchronised; an exception thrown mid set-up may leave copies queued.
    if (stream) cudaStreamSynchronize(stream);
    if (aux) cudaStreamSynchronize(aux);
    mem.free_all();  // stream-ordered frees need the stream
    if (comm && g_comm_destroy) g_comm_destroy(comm);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (h_ctl) pinned_ctl_pool().put(h_ctl);
    if (aux) cudaStreamDestroy(aux);
    if (stream) cudaStreamDestroy(stream);
  }

  int grid_for(long threads) const {
    return static_cast<int>(std::max<long>(1, std::min<long>((threads + pfe_dev::kBlock - 1) / pfe_dev::kBlock, max_grid)));
  }
  int tpv() const { return d == 16 ? 4 : ((d == 2 || d == 4 || d == 8) ? d / 2 : 1); }  // pfe_dev::Cols<d>::TPV
  pfe_host::Launch lv() const { return {grid_for(static_cast<long>(n) * tpv()), stream, sm}; }  // vertex kernels
  pfe_host::Launch le() const { return {grid_for(static_cast<long>(n) * d), stream, sm}; }     // elementwise
  pfe_host::Launch lr() const { return {grid_for(n), stream, sm}; }                            // row kernels

  void ensure_log(long extra) {
    const long need = inner_launched + extra;
    if (need <= log_cap) return;
    long cap = std::max<long>(need, 2 * log_cap + 256);
    int* it = mem.alloc<int>(static_cast<size_t>(cap) * d);
    int* st = mem.alloc<int>(static_cast<size_t>(cap) * d);
    double* rl = mem.alloc<double>(static_cast<size_t>(cap) * d);
    if (log_cap > 0) {
      CK(cudaMemcpyAsync(it, log_it, sizeof(int) * log_cap * d, cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(st, log_st, sizeof(int) * log_cap * d, cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(rl, log_rel, sizeof(double) * log_cap * d, cudaMemcpyDeviceToDevice, stream));
      CK(cudaStreamSynchronize(stream));
      mem.release(log_it);
      mem.release(log_st);
      mem.release(log_rel);
    }
    log_it = it;
    log_st = st;
    log_rel = rl;
    log_cap = cap;
    struct {
      int* a;
      int* b;
      double* c;
    } ptrs{it, st, rl};
    const int capi = static_cast<int>(std::min<long>(cap, 0x7fffffffL));
    CK(cudaMemcpyAsync(&ctl->log_cap, &capi, sizeof(int), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(&ctl->log_iters, &ptrs, sizeof(ptrs), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
  }

  void read_ctl() {
    CK(cudaMemcpyAsync(h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }
};

struct pfe_state {
  pfe_solver* s = nullptr;
  int device = -1;  // a state may outlive its solver; it frees on this device
  DevPool mem;
  double* ybuf[2] = {nullptr, nullptr};  // the two Y allocations (y / y2 alternate between them)
  double *y = nullptr, *y2 = nullptr, *p = nullptr, *breg = nullptr, *rq = nullptr, *r = nullptr;
  double *pb[2] = {nullptr, nullptr}, *q = nullptr;
  double *eb[2] = {nullptr, nullptr}, *es = nullptr;
  double* y0 = nullptr;    // device copy of the initial embedding (pfe_state_reset)
  double* yout = nullptr;  // outer-loop y_old (relative-change test), lazily allocated
  int eb_cur = 0;
  bool inner_zero = true;  // split_b == split_s == 0
  bool rq_valid = false;   // rq == (r/2) sqrt(D) (P - B) for the current P, B
  GraphCache graphs;
};

namespace {

// ------------------------------------------------------------- set-up -----

// Off-diagonal entries of A per forward stencil slot, exactly as
// form_normal_matrix forms them ((hl * (+w)) * (-w) == -((hl * w) * w),
// sparse.cpp:114); +0.0 marks an absent edge (Grid::cf).
// Grid topology on the device (pixel-grid graphs): the forward stencil slot
// of every edge (i, j) -- exactly the host test below: lexicographic order,
// (dy, dx) from j - i, no wrap-around -- written as slot weights wf[i*S + s]
// and the edge -> slot map; any edge that breaks the grid contract sets
// *bad (the host then builds the general CSR topology instead).
// (voff: first vertex of the sub-grid the slot arrays describe, 0 for the
// whole image; row bands pass the edges of their rows only.  slot may be null.)
__global__ void k_grid_slots(long m, int gw, int grad, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                             const double* __restrict__ w, double* __restrict__ wf, int32_t* __restrict__ slot,
                             int* __restrict__ bad, int voff = 0) {
  const int S_ = grad == 1 ? 4 : 12;
  for (long k = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += static_cast<long>(gridDim.x) * blockDim.x) {
    const int i = __ldg(ei + k) - voff, j = __ldg(ej + k) - voff;
    bool ok = true;
    if (k > 0) {
      const int pi = __ldg(ei + k - 1), pj = __ldg(ej + k - 1);
      ok = pi < i || (pi == i && pj < j);
    }
    const long dlt = static_cast<long>(j) - i;
    const int dy = static_cast<int>((dlt + grad) / gw);
    const int dx = static_cast<int>(dlt - static_cast<long>(dy) * gw);
    const int xi = i % gw;
    int s = -1;
    if (xi + dx >= 0 && xi + dx < gw) {
      if (grad == 1) {
        if (dy == 0 && dx == 1) s = 0;
        else if (dy == 1 && dx >= -1 && dx <= 1) s = 2 + dx;
      } else {
        if (dy == 0 && (dx == 1 || dx == 2)) s = dx - 1;
        else if (dy == 1 && dx >= -2 && dx <= 2) s = 4 + dx;
        else if (dy == 2 && dx >= -2 && dx <= 2) s = 9 + dx;
      }
    }
    if (!ok || s < 0) {
      atomicOr(bad, 1);
      continue;
    }
    const int32_t row = i * S_ + s;
    if (slot) slot[k] = row;
    wf[row] = __ldg(w + k);
  }
}

// sqrt(d_v) (correctly rounded, as std::sqrt)
__global__ void k_sqrt(long n, const double* __restrict__ a, double* __restrict__ out) {
  for (long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += static_cast<long>(gridDim.x) * blockDim.x)
    out[v] = sqrt(__ldg(a + v));
}

// diag(A)_v = sum over incident edges in edge-index order (backward slots,
// u ascending, then forward slots; absent slots hold 0 and add +0.0) of
// (hl w) w, then + (r/2) d_v last (sparse.cpp:96-122); inv diag (pcg.cpp:15-20).
// The same operations in the same order as the host loop.
__global__ void k_grid_diag(int gh, int gw, int grad, double hl, double dterm, int precond_none,
                            const double* __restrict__ wf, const double* __restrict__ deg, double* __restrict__ diag,
                            double* __restrict__ invd) {
  const int S_ = grad == 1 ? 4 : 12;
  const long n = static_cast<long>(gh) * gw;
  for (long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += static_cast<long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(v / gw), x = static_cast<int>(v - static_cast<long>(y) * gw);
    double acc = 0.0;
    for (int s = S_ - 1; s >= 0; --s) {
      const int sdy = grad == 1 ? (s == 0 ? 0 : 1) : (s < 2 ? 0 : (s < 7 ? 1 : 2));
      const int sdx = grad == 1 ? (s == 0 ? 1 : s - 2) : (s < 2 ? s + 1 : (s < 7 ? s - 4 : s - 9));
      const int yy = y - sdy, xx = x - sdx;
      if (yy < 0 || xx < 0 || xx >= gw) continue;
      const double w = wf[(v - (static_cast<long>(sdy) * gw + sdx)) * S_ + s];
      acc += (hl * w) * w;
    }
    for (int s = 0; s < S_; ++s) {
      const double w = wf[v * S_ + s];
      acc += (hl * w) * w;
    }
    const double dv = acc + dterm * __ldg(deg + v);
    diag[v] = dv;
    invd[v] = precond_none ? 1.0 : (dv > 0.0 ? 1.0 / dv : 1.0);
  }
}

__global__ void k_grid_coef(long cnt, const double* __restrict__ wf, double hl, double* __restrict__ cf) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double w = wf[i];
    cf[i] = w != 0.0 ? -((hl * w) * w) : 0.0;
  }
}

// --------------------------------------------------- IC(0) preconditioner --
// z = (L L^T)^-1 r with the reference's triangular solves (sparse.cpp:205-238),
// level-scheduled: rows of one level are independent.  One block per
// embedding column walks the levels with a block barrier in between (the
// column's whole dependency chain stays inside one SM).  Forward: row i in
// ascending column order, acc -= L_ik z_k, z_i = acc / L_ii.  Backward (the
// reference scatters column i of L^T after dividing): z_j = (z_j - sum over
// rows i > j in DESCENDING i of L_ij z_i) / L_jj -- the same subtractions in
// the same order, gathered.

// One sweep.  Everything a slot needs that does not depend on z (its row,
// length, diagonal and up to kIcPre entries) is loaded for the next level
// while the current one computes, so a level costs one barrier plus the z
// gathers of its rows (L1: the same block wrote them).
constexpr int kIcPre = 8;
template <int D>
__device__ __forceinline__ void ic_sweep(const IcSweep& sw, const double* src, double* z, int c) {
  struct Pre {
    int pos, beg, len;
    double dg;
    int col[kIcPre];
    double val[kIcPre];
  };
  auto fetch = [&](int t, Pre& p) {
    p.pos = -1;
    if (t < 0) return;
    p.pos = sw.spos[t];
    p.beg = sw.sbeg[t];
    p.len = sw.slen[t];
    p.dg = sw.sdg[t];
#pragma unroll
    for (int e = 0; e < kIcPre; ++e)
      if (e < p.len) {
        p.col[e] = sw.ecol[p.beg + e];
        p.val[e] = sw.eval[p.beg + e];
      }
  };
  auto solve = [&](const Pre& p) {
    double acc = src[static_cast<long>(p.pos) * D + c];
#pragma unroll
    for (int e = 0; e < kIcPre; ++e)
      if (e < p.len) acc -= p.val[e] * z[static_cast<long>(p.col[e]) * D + c];
    for (int e = kIcPre; e < p.len; ++e)
      acc -= sw.eval[p.beg + e] * z[static_cast<long>(sw.ecol[p.beg + e]) * D + c];
    z[static_cast<long>(p.pos) * D + c] = acc / p.dg;
  };
  Pre cur, nxt;
  fetch(sw.nl > 0 && threadIdx.x < sw.lev[1] - sw.lev[0] ? sw.lev[0] + static_cast<int>(threadIdx.x) : -1, cur);
  for (int l = 0; l < sw.nl; ++l) {
    const int b = sw.lev[l], e = sw.lev[l + 1];
    if (l + 1 < sw.nl) {
      const int t = sw.lev[l + 1] + static_cast<int>(threadIdx.x);
      fetch(t < sw.lev[l + 2] ? t : -1, nxt);
    }
    if (cur.pos >= 0) solve(cur);
    for (int t = b + static_cast<int>(threadIdx.x) + blockDim.x; t < e; t += blockDim.x) {  // wide levels
      Pre p;
      fetch(t, p);
      solve(p);
    }
    __syncthreads();
    cur = nxt;
    nxt.pos = -1;
  }
}

// z = (L L^T)^-1 r: forward sweep r -> z, backward sweep in place.
template <int D>
__global__ void __launch_bounds__(256) k_ic_apply(IcDev ic, const double* __restrict__ r, double* z) {
  const int c = blockIdx.x;
  ic_sweep<D>(ic.fwd, r, z, c);
  ic_sweep<D>(ic.bwd, z, z, c);
}

// tot[slot * D + j] = sum_v r_vj z_vj (pcg.cpp:66 / 85 with z = M^-1 r):
// deterministic block partials, reduced by the last block.
template <int D>
__global__ void __launch_bounds__(256) k_ic_dot(int n, const double* __restrict__ r, const double* __restrict__ z,
                                                double* part, pfe_dev::Ctl* ctl, double* tot) {
  double acc[1][D] = {};
  for (long v = blockIdx.x * 256L + threadIdx.x; v < n; v += static_cast<long>(gridDim.x) * 256) {
#pragma unroll
    for (int c = 0; c < D; ++c) acc[0][c] += r[v * D + c] * z[v * D + c];
  }
  pfe_dev::block_reduce_store<1, D, D, 256>(acc, part);
  __shared__ double out[1][D];
  if (pfe_dev::grid_reduce_last<1, D, 256>(part, ctl, out) && threadIdx.x < D) tot[threadIdx.x] = out[0][threadIdx.x];
}

template <int D>
void ic_apply_d(const IcDev& ic, const double* r, double* z, cudaStream_t s) {
  k_ic_apply<D><<<D, 256, 0, s>>>(ic, r, z);
}
template <int D>
void ic_dot_d(int n, const double* r, const double* z, double* part, pfe_dev::Ctl* ctl, double* tot, int grid,
              cudaStream_t s) {
  k_ic_dot<D><<<grid, 256, 0, s>>>(n, r, z, part, ctl, tot);
}
template <int... Ds>
void ic_apply_dispatch(int d, std::integer_sequence<int, Ds...>, const IcDev& ic, const double* r, double* z,
                       cudaStream_t s) {
  ((d == Ds + 1 ? ic_apply_d<Ds + 1>(ic, r, z, s) : void()), ...);
}
template <int... Ds>
void ic_dot_dispatch(int d, std::integer_sequence<int, Ds...>, int n, const double* r, const double* z, double* part,
                     pfe_dev::Ctl* ctl, double* tot, int grid, cudaStream_t s) {
  ((d == Ds + 1 ? ic_dot_d<Ds + 1>(n, r, z, part, ctl, tot, grid, s) : void()), ...);
}

struct HostGraph {
  int n;
  long m;
  const int32_t* ei;
  const int32_t* ej;
  const double* w;
  const double* deg;
};

// Validation in the reference's order: difference_matrix/csr_from_triplets
// (sparse.cpp:12-21), form_normal_matrix (98-106), PcgOperator (pcg.cpp:10-12),
// PfeSolver (solver.cpp:51-57).
void validate(const HostGraph& g, const pfe_params& p, bool check_solver_caps) {
  if (g.n < 1) config_error("graph: n must be >= 1");
  if (g.m < 0) config_error("graph: negative edge count");
  // first offending edge found in parallel, then reported by the serial
  // checks below in the reference's order
  std::atomic<long> first_bad{g.m};
  parallel_for(g.m, [&](long b, long e) {
    for (long k = b; k < e; ++k) {
      const int i = g.ei[k], j = g.ej[k];
      if (i < 0 || i >= g.n || j < 0 || j >= g.n || !std::isfinite(g.w[k]) || i >= j) {
        long cur = first_bad.load();
        while (k < cur && !first_bad.compare_exchange_weak(cur, k)) {
        }
        return;
      }
    }
  });
  for (long k = first_bad.load(); k < g.m; ++k) {
    const int i = g.ei[k], j = g.ej[k];
    if (i < 0 || i >= g.n || j < 0 || j >= g.n)
      config_error("csr_from_triplets: entry (" + std::to_string(k) + "," + std::to_string(i < 0 || i >= g.n ? i : j) +
                   ") outside " + std::to_string(g.m) + "x" + std::to_string(g.n));
    if (!std::isfinite(g.w[k])) config_error("csr_from_triplets: non-finite value");
    if (i >= j) config_error("graph: edge " + std::to_string(k) + " must satisfy i < j (graph.hpp:15-17)");
  }
  if (!g.deg) config_error("form_normal_matrix: degree size mismatch");
  if (p.lambda < 0.0) config_error("form_normal_matrix: lambda must be >= 0");
  if (p.r <= 0.0) config_error("form_normal_matrix: r must be > 0");
  {
    // first offending vertex, found in parallel (16.8 M vertices on C4)
    std::atomic<long> bad_deg{g.n};
    parallel_for(g.n, [&](long b, long e) {
      for (long v = b; v < e; ++v)
        if (!(g.deg[v] > 0.0)) {
          long cur = bad_deg.load();
          while (v < cur && !bad_deg.compare_exchange_weak(cur, v)) {
          }
          return;
        }
    });
    if (bad_deg.load() < g.n)
      config_error("form_normal_matrix: nonpositive degree at vertex " + std::to_string(bad_deg.load()) +
                   " (isolated vertex)");
  }
  if (p.pcg_rel_tol <= 0.0) config_error("PcgOperator: rel_tol must be > 0");
  if (p.pcg_max_iter < 1) config_error("PcgOperator: max_iter must be >= 1");
  if (p.dim < 1) config_error("PfeSolver: dim must be >= 1");
  if (p.lambda <= 0.0 || p.r <= 0.0) config_error("PfeSolver: lambda and r must be > 0");
  if (check_solver_caps && (p.soc_max < 1 || p.sb_max_stage1 < 1))
    config_error("PfeSolver: iteration caps must be >= 1");
  if (p.dim > pfe_dev::kMaxD) config_error("PfeSolver: the B200 kernels support dim <= 16");
  if (p.preconditioner < 0 || p.preconditioner > 2) config_error("PcgConfig: unknown preconditioner");
}

// Forward stencil slot of edge (i, j) for a W-wide grid of radius R, or -1.
int grid_slot(int R, int W, int i, int j) {
  const int yi = i / W, xi = i % W, yj = j / W, xj = j % W;
  const int dy = yj - yi, dx = xj - xi;
  if (R == 1) {
    if (dy == 0 && dx == 1) return 0;
    if (dy == 1 && dx >= -1 && dx <= 1) return 2 + dx;
    return -1;
  }
  if (dy == 0 && (dx == 1 || dx == 2)) return dx - 1;
  if (dy == 1 && dx >= -2 && dx <= 2) return 4 + dx;
  if (dy == 2 && dx >= -2 && dx <= 2) return 9 + dx;
  return -1;
}

// Breadth-first order of the vertices (components in vertex order, neighbours
// in incidence order): perm[v] = position of v.  Used as the storage order of
// general graphs and as the basis of vertex-range partitions.
// Reverse Cuthill-McKee alternative (A/B experiments, PFE_STORAGE_ORDER=rcm):
// per component, BFS from a minimum-degree vertex with each vertex's
// unvisited neighbours taken in ascending degree, then the whole order
// reversed.  Aims at a smaller bandwidth than the plain BFS.
std::vector<int> rcm_storage_order(int n, const std::vector<int>& iptr, const int* inbr) {
  std::vector<int> perm(n, -1), order;
  order.reserve(n);
  std::vector<int> deg(n), byd(n);
  for (int v = 0; v < n; ++v) deg[v] = iptr[v + 1] - iptr[v];
  std::iota(byd.begin(), byd.end(), 0);
  std::stable_sort(byd.begin(), byd.end(), [&](int a, int b) { return deg[a] < deg[b]; });
  std::vector<char> seen(n, 0);
  std::vector<int> nb;
  for (int s0 : byd) {
    if (seen[s0]) continue;
    size_t head = order.size();
    seen[s0] = 1;
    order.push_back(s0);
    while (head < order.size()) {
      const int v = order[head++];
      nb.clear();
      for (int k = iptr[v]; k < iptr[v + 1]; ++k)
        if (!seen[inbr[k]]) {
          seen[inbr[k]] = 1;
          nb.push_back(inbr[k]);
        }
      std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
      order.insert(order.end(), nb.begin(), nb.end());
    }
  }
  for (int i = 0; i < n; ++i) perm[order[n - 1 - i]] = i;
  return perm;
}

// Breadth-first storage order (serial queue: a level-parallel version that
// reproduced the same order with atomic first-visit keys measured slower on
// C5, 217 vs 130 ms).
std::vector<int> bfs_storage_order(int n, const std::vector<int>& iptr, const int* inbr) {
  if (const char* o = std::getenv("PFE_STORAGE_ORDER"); o && std::string(o) == "rcm")
    return rcm_storage_order(n, iptr, inbr);
  std::vector<int> perm(n, -1), queue(n);
  int next = 0, head = 0;
  for (int s0 = 0; s0 < n; ++s0) {
    if (perm[s0] >= 0) continue;
    perm[s0] = next;
    queue[next++] = s0;
    while (head < next) {
      const int v = queue[head++];
      for (int k = iptr[v]; k < iptr[v + 1]; ++k) {
        const int u = inbr[k];
        if (perm[u] < 0) {
          perm[u] = next;
          queue[next++] = u;
        }
      }
    }
  }
  return perm;
}


// Incidence lists in increasing edge index (the row order of M^T).
struct Incidence {
  std::vector<int> iptr;
  uvec<int> inbr, ieid;
  uvec<double> iw;
};
Incidence build_incidence(const HostGraph& g) {
  Incidence c;
  const int n = g.n;
  const long m = g.m;
  c.iptr.assign(static_cast<size_t>(n) + 1, 0);
  c.inbr.resize(static_cast<size_t>(2 * m));
  c.ieid.resize(static_cast<size_t>(2 * m));
  c.iw.resize(static_cast<size_t>(2 * m));
  // counting sort by vertex, edges kept in increasing index: T threads own
  // consecutive edge chunks; per-thread counts give each thread its slots
  const long hw = std::max(1u, std::thread::hardware_concurrency());
  long T = std::min<long>(std::min<long>(hw, 16), std::max(1L, m / (1L << 18)));
  T = std::max(1L, std::min<long>(T, (256L << 20) / (4L * std::max(1, n))));  // counts memory cap
  const long per = (m + T - 1) / T;
  std::vector<int> cnt(static_cast<size_t>(T) * n, 0);
  auto run = [&](auto&& body) {
    std::vector<std::thread> pool;
    for (long t = 0; t < T; ++t) pool.emplace_back([&, t] { body(t, t * per, std::min(m, (t + 1) * per)); });
    for (auto& th : pool) th.join();
  };
  run([&](long t, long kb, long ke) {
    int* ct = cnt.data() + t * n;
    for (long k = kb; k < ke; ++k) {
      ++ct[g.ei[k]];
      ++ct[g.ej[k]];
    }
  });
  for (int v = 0; v < n; ++v) {
    int tot = 0;
    for (long t = 0; t < T; ++t) tot += cnt[static_cast<size_t>(t) * n + v];
    c.iptr[v + 1] = c.iptr[v] + tot;
  }
  parallel_for(n, [&](long vb, long ve) {  // counts -> each thread's first slot per vertex
    for (long v = vb; v < ve; ++v) {
      int base = c.iptr[v];
      for (long t = 0; t < T; ++t) {
        int& x = cnt[static_cast<size_t>(t) * n + v];
        const int k = x;
        x = base;
        base += k;
      }
    }
  });
  run([&](long t, long kb, long ke) {
    int* fill = cnt.data() + t * n;
    for (long k = kb; k < ke; ++k) {
      const int i = g.ei[k], j = g.ej[k];
      int at = fill[i]++;
      c.inbr[at] = j;
      c.ieid[at] = static_cast<int>(k);
      c.iw[at] = g.w[k];
      at = fill[j]++;
      c.inbr[at] = i;
      c.ieid[at] = static_cast<int>(k);
      c.iw[at] = g.w[k];
    }
  });
  return c;
}

// A = (lambda/2) M^T M + (r/2) D in the reference's natural row order: rows
// sorted by column, duplicate columns summed in edge order, exact zeros
// dropped (csr_from_triplets over form_normal_matrix's triplets,
// sparse.cpp:96-122).  `diag` holds the finished diagonal per vertex.
void natural_rows(int n, const Incidence& inc, double hl, const double* diag, std::vector<int>& nptr,
                  std::vector<int>& ncol, std::vector<double>& nval) {
  nptr.assign(static_cast<size_t>(n) + 1, 0);
  ncol.clear();
  nval.clear();
  ncol.reserve(inc.inbr.size() + n);
  nval.reserve(inc.inbr.size() + n);
  std::vector<std::pair<int, double>> row;
  for (int v = 0; v < n; ++v) {
    row.clear();
    for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) row.emplace_back(inc.inbr[k], -((hl * inc.iw[k]) * inc.iw[k]));
    row.emplace_back(v, diag[v]);
    std::stable_sort(row.begin(), row.end(),
                     [](const std::pair<int, double>& a, const std::pair<int, double>& b) { return a.first < b.first; });
    for (size_t t = 0; t < row.size();) {
      const int col = row[t].first;
      double s = 0.0;
      if (col == v) {
        s = row[t].second;
        ++t;
      } else {
        for (; t < row.size() && row[t].first == col; ++t) s += row[t].second;
      }
      if (s != 0.0) {
        ncol.push_back(col);
        nval.push_back(s);
      }
    }
    nptr[v + 1] = static_cast<int>(ncol.size());
  }
}

// Builds the device topology.  Diagonal of A: sum over incident edges in
// edge order of (hl * w) * w, then + (0.5 r) deg_v last — the accumulation
// order csr_from_triplets applies to form_normal_matrix's triplets.
double* grid_coef(pfe_solver* S, const double* dwf, long cnt, double hl, cudaStream_t st) {
  double* dcf = S->mem.alloc<double>(static_cast<size_t>(cnt));
  const int grid = static_cast<int>(std::min<long>(4L * S->sm * 8, (cnt + 255) / 256));
  if (cnt > 0) k_grid_coef<<<std::max(1, grid), 256, 0, st>>>(cnt, dwf, hl, dcf);
  CK(cudaGetLastError());
  return dcf;
}

// IC(0) factor of A in the reference's (natural) row order, its level
// schedules and device copy (columns as storage positions).  A factor that
// breaks down after every shift falls back to Jacobi like the reference.
void build_ic(pfe_solver* S, int n, const std::vector<int>& aptr, const std::vector<int>& acol,
              const std::vector<double>& aval, const std::vector<int>& perm) {
  pfe_host::IcFactorHost f;
  if (!pfe_host::ic0_factor(n, aptr.data(), acol.data(), aval.data(), f)) {
    S->ic = false;
    S->jacobi_fallback = true;
    return;
  }
  auto by_level = [n](const std::vector<int>& lev, int nl, std::vector<int>& rows, std::vector<int>& off) {
    off.assign(static_cast<size_t>(nl) + 1, 0);
    for (int i = 0; i < n; ++i) ++off[lev[i] + 1];
    for (int l = 0; l < nl; ++l) off[l + 1] += off[l];
    rows.assign(static_cast<size_t>(n), 0);
    std::vector<int> fill(off.begin(), off.end() - 1);
    for (int i = 0; i < n; ++i) rows[fill[lev[i]]++] = i;
  };
  // forward levels: 1 + the deepest column a row reads
  std::vector<int> lev(static_cast<size_t>(n), 0);
  int nlf = 0;
  for (int i = 0; i < n; ++i) {
    int l = 0;
    for (int k = f.ptr[i]; k < f.ptr[i + 1] - 1; ++k) l = std::max(l, lev[f.idx[k]] + 1);
    lev[i] = l;
    nlf = std::max(nlf, l + 1);
  }
  std::vector<int> frows, flev;
  by_level(lev, nlf, frows, flev);
  // backward: below-diagonal entries of column j, rows descending; levels
  // from the columns of L (a column waits for every row that updates it)
  std::vector<int> bptr(static_cast<size_t>(n) + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int k = f.ptr[i]; k < f.ptr[i + 1] - 1; ++k) ++bptr[f.idx[k] + 1];
  for (int j = 0; j < n; ++j) bptr[j + 1] += bptr[j];
  std::vector<int> brow(static_cast<size_t>(bptr[n])), bfill(bptr.begin(), bptr.end() - 1);
  std::vector<double> bval(static_cast<size_t>(bptr[n]));
  std::vector<int> blv(static_cast<size_t>(n), 0);
  int nlb = 0;
  for (int i = n - 1; i >= 0; --i) {
    nlb = std::max(nlb, blv[i] + 1);
    for (int k = f.ptr[i]; k < f.ptr[i + 1] - 1; ++k) {
      const int j = f.idx[k];
      brow[bfill[j]] = i;
      bval[bfill[j]++] = f.val[k];
      blv[j] = std::max(blv[j], blv[i] + 1);
    }
  }
  std::vector<int> brows, blev;
  by_level(blv, nlb, brows, blev);
  // level-ordered slots with their entries laid out contiguously
  cudaStream_t st = S->stream;
  auto upload_sweep = [&](const std::vector<int>& rows, const std::vector<int>& levs, int nl, auto&& row_entries,
                          auto&& row_diag, IcSweep& out) {
    std::vector<int> spos(static_cast<size_t>(n)), sbeg(static_cast<size_t>(n)), slen(static_cast<size_t>(n)), ecol;
    std::vector<double> sdg(static_cast<size_t>(n)), ev;
    for (int t = 0; t < n; ++t) {
      const int i = rows[t];
      spos[t] = perm[i];
      sbeg[t] = static_cast<int>(ecol.size());
      row_entries(i, ecol, ev);
      slen[t] = static_cast<int>(ecol.size()) - sbeg[t];
      sdg[t] = row_diag(i);
    }
    out.spos = S->mem.upload(spos, st);
    out.sbeg = S->mem.upload(sbeg, st);
    out.slen = S->mem.upload(slen, st);
    out.sdg = S->mem.upload(sdg, st);
    out.ecol = S->mem.upload(ecol, st);
    out.eval = S->mem.upload(ev, st);
    out.lev = S->mem.upload(levs, st);
    out.nl = nl;
    CK(cudaStreamSynchronize(st));  // the host vectors die here
  };
  // forward row i: L_ik, k < i, ascending columns (sparse.cpp:209-218)
  upload_sweep(
      frows, flev, nlf,
      [&](int i, std::vector<int>& ec, std::vector<double>& ev) {
        for (int k = f.ptr[i]; k < f.ptr[i + 1] - 1; ++k) {
          ec.push_back(perm[f.idx[k]]);
          ev.push_back(f.val[k]);
        }
      },
      [&](int i) { return f.val[f.ptr[i + 1] - 1]; }, S->icd.fwd);
  // backward column j: L_ij, i > j, descending rows (sparse.cpp:225-236)
  upload_sweep(
      brows, blev, nlb,
      [&](int j, std::vector<int>& ec, std::vector<double>& ev) {
        for (int k = bptr[j]; k < bptr[j + 1]; ++k) {
          ec.push_back(perm[brow[k]]);
          ev.push_back(bval[k]);
        }
      },
      [&](int j) { return f.val[f.ptr[j + 1] - 1]; }, S->icd.bwd);
  S->zbuf = S->mem.alloc<double>(static_cast<size_t>(n) * S->d);
}

void build_topology(pfe_solver* S, const HostGraph& g, int gh, int gw, int grad) {
  const int n = g.n;
  const long m = g.m;
  const double hl = 0.5 * S->prm.lambda;
  const double dterm = 0.5 * S->prm.r;
  cudaStream_t st = S->stream;

  auto finish_diag = [&](std::vector<double>& diag) {
    std::vector<double> invd(n);
    parallel_for(n, [&](long b, long e) {
      for (long v = b; v < e; ++v) {
        diag[v] += dterm * g.deg[v];  // the (r/2) d_v triplet is summed last
        invd[v] = S->prm.preconditioner == PFE_PRECOND_NONE ? 1.0 : (diag[v] > 0.0 ? 1.0 / diag[v] : 1.0);
      }
    });
    S->diag = S->mem.upload(diag, st);
    S->invd = S->mem.upload(invd, st);
  };

  // grid eligibility: hint consistent, W wide enough for the slot order to be
  // the column order, edges strictly lexicographic and all stencil offsets.
  bool grid = gh > 0 && gw > 0 && static_cast<long>(gh) * gw == n && (grad == 1 || grad == 2) &&
              gw >= 2 * grad + 2;
  if (grid && static_cast<long>(n) * (grad == 1 ? 4 : 12) < 0x7fffffffL &&
      !(std::getenv("PFE_HOST_TOPOLOGY") && std::getenv("PFE_HOST_TOPOLOGY")[0] == '1')) {
    // Pixel grid on the device: upload the edge list once, derive the slot
    // weights, the edge -> slot map, diag and inv diag there (the host loop
    // below costs ~0.4 s on C4's 67 M edges and uploads the same bytes).
    const int S_ = grad == 1 ? 4 : 12;
    const long ns = static_cast<long>(n) * S_;
    DevPool tmp;
    tmp.stream = tmp.fstream = st;
    int32_t* d_ei = tmp.alloc<int32_t>(static_cast<size_t>(m));
    int32_t* d_ej = tmp.alloc<int32_t>(static_cast<size_t>(m));
    double* d_w = tmp.alloc<double>(static_cast<size_t>(m));
    double* d_deg = S->mem.alloc<double>(static_cast<size_t>(n));  // kept: the solver's degree array
    int* d_bad = tmp.alloc<int>(1);
    copy_h2d(d_ei, g.ei, sizeof(int32_t) * m, st);
    copy_h2d(d_ej, g.ej, sizeof(int32_t) * m, st);
    copy_h2d(d_w, g.w, sizeof(double) * m, st);
    copy_h2d(d_deg, g.deg, sizeof(double) * n, st);
    double* dwf = S->mem.alloc<double>(static_cast<size_t>(ns));
    int32_t* dslot = S->mem.alloc<int32_t>(static_cast<size_t>(std::max(m, 1L)));
    CK(cudaMemsetAsync(dwf, 0, sizeof(double) * ns, st));
    CK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    const int blocks = static_cast<int>(std::min<long>(std::max<long>(1, (m + 255) / 256), 32L * S->sm));
    if (m > 0) k_grid_slots<<<blocks, 256, 0, st>>>(m, gw, grad, d_ei, d_ej, d_w, dwf, dslot, d_bad);
    CK(cudaGetLastError());
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!bad) {
      if (S->row_hi < 0) {
        S->row_lo = 0;
        S->row_hi = gh;
      }
      S->diag = S->mem.alloc<double>(static_cast<size_t>(n));
      S->invd = S->mem.alloc<double>(static_cast<size_t>(n));
      const int vb = static_cast<int>(std::min<long>((n + 255) / 256, 32L * S->sm));
      k_grid_diag<<<std::max(1, vb), 256, 0, st>>>(gh, gw, grad, hl, dterm, S->prm.preconditioner == PFE_PRECOND_NONE,
                                                   dwf, d_deg, S->diag, S->invd);
      CK(cudaGetLastError());
      S->d_edge_slot = dslot;
      S->edge_rows = ns;
      S->deg = d_deg;  // grids keep vertex order: upload_degree has nothing left to do
      S->sqd = S->mem.alloc<double>(static_cast<size_t>(n));
      k_sqrt<<<std::max(1, vb), 256, 0, st>>>(n, d_deg, S->sqd);
      CK(cudaGetLastError());
      double* dcf = grid_coef(S, dwf, ns, hl, st);
      CK(cudaStreamSynchronize(st));  // the temporaries are freed next
      tmp.free_all();
      if (grad == 1) {
        S->topo.kind = pfe_host::kTopoGrid1;
        S->topo.g1 = pfe_dev::Grid<1>{n, gh, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
        S->topo.g1.cf = dcf;
      } else {
        S->topo.kind = pfe_host::kTopoGrid2;
        S->topo.g2 = pfe_dev::Grid<2>{n, gh, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
        S->topo.g2.cf = dcf;
      }
      return;
    }
    tmp.free_all();
    S->mem.release(dwf);
    S->mem.release(dslot);
    S->mem.release(d_deg);
    grid = false;  // not a stencil graph after all: general CSR topology
  }
  std::vector<long> slot_of;
  if (grid) {
    slot_of.resize(static_cast<size_t>(m));
    const int S_ = grad == 1 ? 4 : 12;
    // j - i identifies (dy, dx) uniquely since |dx| <= R < W / 2; the column
    // of i rules out wrap-around
    std::atomic<bool> ok{true};
    parallel_for(m, [&](long kb, long ke) {
    int cur_i = -1, xi = 0;
    for (long k = kb; k < ke; ++k) {
      const int i = g.ei[k], j = g.ej[k];
      if (k > 0 && !(g.ei[k - 1] < i || (g.ei[k - 1] == i && g.ej[k - 1] < j))) {
        ok = false;
        return;
      }
      if (i != cur_i) {
        xi = i % gw;
        cur_i = i;
      }
      const long dlt = static_cast<long>(j) - i;
      const int dy = static_cast<int>((dlt + grad) / gw);
      const int dx = static_cast<int>(dlt - static_cast<long>(dy) * gw);
      int s = -1;
      if (xi + dx >= 0 && xi + dx < gw) {
        if (grad == 1) {
          if (dy == 0 && dx == 1) s = 0;
          else if (dy == 1 && dx >= -1 && dx <= 1) s = 2 + dx;
        } else {
          if (dy == 0 && (dx == 1 || dx == 2)) s = dx - 1;
          else if (dy == 1 && dx >= -2 && dx <= 2) s = 4 + dx;
          else if (dy == 2 && dx >= -2 && dx <= 2) s = 9 + dx;
        }
      }
      if (s < 0) {
        ok = false;
        return;
      }
      slot_of[k] = static_cast<long>(i) * S_ + s;
    }
    });
    grid = ok.load();
  }
  if (grid) {
    const int S_ = grad == 1 ? 4 : 12;
    if (S->row_hi < 0) {
      S->row_lo = 0;
      S->row_hi = gh;
    }
    uvec<double> wf(static_cast<size_t>(n) * S_);  // zero-filled in parallel: absent slots stay 0
    parallel_for(static_cast<long>(wf.size()), [&](long b, long e) { std::fill(wf.begin() + b, wf.begin() + e, 0.0); });
    parallel_for(m, [&](long b, long e) {
      for (long k = b; k < e; ++k) wf[static_cast<size_t>(slot_of[k])] = g.w[k];
    });
    // diag(A)_v: incident edges in edge-index order = backward slots (u
    // ascending) then forward slots; absent slots hold 0 and add +0.0.
    std::vector<double> diag(n, 0.0);
    int off[12], sdy[12], sdx[12];
    for (int s = 0; s < S_; ++s) {
      sdy[s] = grad == 1 ? (s == 0 ? 0 : 1) : (s < 2 ? 0 : (s < 7 ? 1 : 2));
      sdx[s] = grad == 1 ? (s == 0 ? 1 : s - 2) : (s < 2 ? s + 1 : (s < 7 ? s - 4 : s - 9));
      off[s] = sdy[s] * gw + sdx[s];
    }
    parallel_for(gh, [&](long yb, long ye) {
    for (int y = static_cast<int>(yb), v = static_cast<int>(yb) * gw; y < ye; ++y) {
      for (int x = 0; x < gw; ++x, ++v) {
        double acc = 0.0;
        for (int s = S_ - 1; s >= 0; --s) {
          const int yy = y - sdy[s], xx = x - sdx[s];
          if (yy < 0 || xx < 0 || xx >= gw) continue;
          const double w = wf[static_cast<size_t>(v - off[s]) * S_ + s];
          acc += (hl * w) * w;
        }
        for (int s = 0; s < S_; ++s) {
          const double w = wf[static_cast<size_t>(v) * S_ + s];
          acc += (hl * w) * w;
        }
        diag[v] = acc;
      }
    }
    }, std::max(1L, (1L << 16) / gw));
    finish_diag(diag);
    double* dwf = S->mem.upload(wf, st);
    S->edge_row = std::move(slot_of);
    S->edge_rows = static_cast<long>(n) * S_;
    double* dcf = grid_coef(S, dwf, static_cast<long>(n) * S_, hl, st);
    if (grad == 1) {
      S->topo.kind = pfe_host::kTopoGrid1;
      S->topo.g1 = pfe_dev::Grid<1>{n, gh, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
      S->topo.g1.cf = dcf;
    } else {
      S->topo.kind = pfe_host::kTopoGrid2;
      S->topo.g2 = pfe_dev::Grid<2>{n, gh, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
      S->topo.g2.cf = dcf;
    }
    return;
  }

  // General graph on the device (pfe_csrbuild.cu): every array derived from
  // the uploaded edge list by kernels, bit-identical to the host builder
  // below.  IC(0) solvers need A on the host (the factor), and graphs with
  // very many components fall through to the host builder.
  {
    const char* sw = std::getenv("PFE_DEVICE_CSR");
    const bool host_only = std::getenv("PFE_HOST_TOPOLOGY") && std::getenv("PFE_HOST_TOPOLOGY")[0] == '1';
    const bool want = sw ? sw[0] == '1' : m >= (1L << 17);
    if (want && !host_only && !S->ic && !(sw && sw[0] == '0')) {
      pfe_host::CsrDevArrays o;
      auto alloc = [](void* ctx, size_t bytes) -> void* {
        return static_cast<pfe_solver*>(ctx)->mem.alloc<char>(bytes);
      };
      auto h2d = [](void* dst, const void* src, size_t bytes, void* stream) {
        copy_h2d(dst, src, bytes, static_cast<cudaStream_t>(stream));
      };
      if (pfe_host::csr_topology_device(n, m, g.ei, g.ej, g.w, g.deg, hl, dterm,
                                        S->prm.preconditioner == PFE_PRECOND_NONE, st, alloc, S, h2d, 4096, &o)) {
        S->diag = o.diag;
        S->invd = o.invd;
        S->deg = o.deg;
        S->sqd = o.sqd;
        S->perm_d = o.perm;
        S->d_edge_slot = o.edge_row;  // the host copy is downloaded on first use (state get / set)
        S->edge_rows = m;
        pfe_dev::Csr c{};
        c.n = n;
        c.vb = 0;
        c.ve = n;
        c.aptr = o.aptr;
        c.acol = o.acol;
        c.aval = o.aval;
        c.iptr = o.iptr;
        c.inbr = o.inbr;
        c.ieid = o.ieid;
        c.iw = o.iw;
        c.invd = S->invd;
        S->topo.kind = pfe_host::kTopoCsr;
        S->topo.csr = c;
        return;
      }
    }
  }

  // incidence lists in increasing edge index (the row order of M^T)
  const bool tmr = [] {
    const char* e = std::getenv("PFE_SETUP_TIMING");
    return e && e[0] == '1';
  }();
  auto tq = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!tmr) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  topology %-10s %.2f ms\n", what, std::chrono::duration<double, std::milli>(t - tq).count());
    tq = t;
  };
  Incidence inc = build_incidence(g);
  mark("incidence");
  const std::vector<int>& iptr = inc.iptr;
  const uvec<int>& inbr = inc.inbr;
  const uvec<int>& ieid = inc.ieid;
  const uvec<double>& iw = inc.iw;
  std::vector<double> diag(n);
  parallel_for(n, [&](long vb, long ve) {
    for (long v = vb; v < ve; ++v) {
      double acc = 0.0;
      for (int k = iptr[v]; k < iptr[v + 1]; ++k) acc += (hl * iw[k]) * iw[k];
      diag[v] = acc;
    }
  }, 4096);
  // storage order: BFS over the incidence graph (components in vertex order),
  // so the rows a vertex gathers sit near its own and stay in L2 / L1
  mark("diag");
  std::vector<int> perm = bfs_storage_order(n, iptr, inbr.data()), inv(n);
  mark("bfs");
  for (int v = 0; v < n; ++v) inv[perm[v]] = v;
  {
    // diag / inv_diag in storage order ((r/2) d_v is added last, as finish_diag does)
    std::vector<double> dperm(n), invd(n);
    for (int v = 0; v < n; ++v) dperm[perm[v]] = diag[v] + dterm * g.deg[v];
    for (int x = 0; x < n; ++x)
      invd[x] = S->prm.preconditioner == PFE_PRECOND_NONE ? 1.0 : (dperm[x] > 0.0 ? 1.0 / dperm[x] : 1.0);
    for (int v = 0; v < n; ++v) diag[v] = dperm[perm[v]];
    S->diag = S->mem.upload(dperm, st);
    S->invd = S->mem.upload(invd, st);
  }

  // General CSR: A rows sorted by column with duplicate columns summed in
  // edge order (stable sort), exact zeros dropped, diagonal in place.  Rows
  // are merged in parallel into an upper-bound layout, then compacted.
  std::vector<long> ub(static_cast<size_t>(n) + 1, 0);
  for (int x = 0; x < n; ++x) {
    const int v = inv[x];
    ub[x + 1] = ub[x] + (iptr[v + 1] - iptr[v]) + 1;
  }
  uvec<int> tcol(static_cast<size_t>(ub[n])), tlen(static_cast<size_t>(n));
  uvec<double> tval(static_cast<size_t>(ub[n]));
  parallel_for(n, [&](long xb, long xe) {
    std::vector<std::pair<int, double>> row;
    for (long x = xb; x < xe; ++x) {
      const int v = inv[x];  // storage row x holds vertex v's row, in the reference's column order
      row.clear();
      for (int k = iptr[v]; k < iptr[v + 1]; ++k) row.emplace_back(inbr[k], -((hl * iw[k]) * iw[k]));
      row.emplace_back(v, diag[v]);
      std::stable_sort(row.begin(), row.end(),
                       [](const std::pair<int, double>& a, const std::pair<int, double>& b) { return a.first < b.first; });
      long at = ub[x];
      for (size_t t = 0; t < row.size();) {
        const int col = row[t].first;
        double s = 0.0;
        if (col == v) {
          s = row[t].second;  // diagonal already accumulated in csr_from_triplets order
          ++t;
        } else {
          for (; t < row.size() && row[t].first == col; ++t) s += row[t].second;
        }
        if (s != 0.0) {
          tcol[static_cast<size_t>(at)] = perm[col];
          tval[static_cast<size_t>(at)] = s;
          ++at;
        }
      }
      tlen[x] = static_cast<int>(at - ub[x]);
    }
  }, 4096);
  mark("rows");
  std::vector<int> aptr(static_cast<size_t>(n) + 1, 0);
  for (int x = 0; x < n; ++x) aptr[x + 1] = aptr[x] + tlen[x];
  uvec<int> acol(static_cast<size_t>(aptr[n]));
  uvec<double> aval(static_cast<size_t>(aptr[n]));
  parallel_for(n, [&](long xb, long xe) {
    for (long x = xb; x < xe; ++x) {
      std::copy(tcol.begin() + ub[x], tcol.begin() + ub[x] + tlen[x], acol.begin() + aptr[x]);
      std::copy(tval.begin() + ub[x], tval.begin() + ub[x] + tlen[x], aval.begin() + aptr[x]);
    }
  }, 4096);
  if (S->ic) {
    // A in the reference's row order (the IC(0) factor depends on it)
    std::vector<int> nptr, ncol;
    std::vector<double> nval;
    natural_rows(n, inc, hl, diag.data(), nptr, ncol, nval);
    build_ic(S, n, nptr, ncol, nval, perm);
  }
  // edge storage follows the vertex storage order: the edges a vertex owns
  // (it is their first endpoint) are consecutive rows of the edge arrays
  mark("compact");
  uvec<int> epos(static_cast<size_t>(m));
  std::vector<int> own(static_cast<size_t>(n) + 1, 0);  // owned-edge offsets in storage order
  parallel_for(n, [&](long xb, long xe) {
    for (long x = xb; x < xe; ++x) {
      const int v = inv[x];
      int c = 0;
      for (int k = iptr[v]; k < iptr[v + 1]; ++k) c += inbr[k] > v ? 1 : 0;
      own[x + 1] = c;
    }
  }, 4096);
  for (int x = 0; x < n; ++x) own[x + 1] += own[x];
  parallel_for(n, [&](long xb, long xe) {
    for (long x = xb; x < xe; ++x) {
      const int v = inv[x];
      int next = own[x];
      for (int k = iptr[v]; k < iptr[v + 1]; ++k)
        if (inbr[k] > v) epos[ieid[k]] = next++;
    }
  }, 4096);
  // incidence lists in storage order: (neighbour row, w, edge row << 1 | [v is
  // the edge's first endpoint]), each in increasing edge index
  std::vector<int> iptr2(static_cast<size_t>(n) + 1, 0);
  uvec<int> inbr2(static_cast<size_t>(2 * m)), ieid2(static_cast<size_t>(2 * m));
  uvec<double> iw2(static_cast<size_t>(2 * m));
  for (int x = 0; x < n; ++x) {
    const int v = inv[x];
    iptr2[x + 1] = iptr2[x] + (iptr[v + 1] - iptr[v]);
  }
  parallel_for(n, [&](long xb, long xe) {
    for (long x = xb; x < xe; ++x) {
      const int v = inv[x];
      int at = iptr2[x];
      for (int k = iptr[v]; k < iptr[v + 1]; ++k, ++at) {
        inbr2[at] = perm[inbr[k]];
        ieid2[at] = (epos[ieid[k]] << 1) | (inbr[k] > v ? 1 : 0);
        iw2[at] = iw[k];
      }
    }
  }, 4096);
  mark("remap");
  S->perm_h = perm;
  S->perm_d = S->mem.upload(perm, st);
  S->edge_row.assign(epos.begin(), epos.end());
  S->edge_rows = m;
  pfe_dev::Csr c{};
  c.n = n;
  c.vb = 0;
  c.ve = n;
  c.aptr = S->mem.upload(aptr, st);
  c.acol = S->mem.upload(acol, st);
  c.aval = S->mem.upload(aval, st);
  c.iptr = S->mem.upload(iptr2, st);
  c.inbr = S->mem.upload(inbr2, st);
  c.ieid = S->mem.upload(ieid2, st);
  c.iw = S->mem.upload(iw2, st);
  c.invd = S->invd;
  S->topo.kind = pfe_host::kTopoCsr;
  S->topo.csr = c;
  mark("upload");
}

void init_common(pfe_solver* S, const pfe_exec* x, int d) {
  S->device = x ? x->device : 0;
  require_device(S->device);
  S->use_graphs = x ? x->use_graphs != 0 : true;
  S->warn = x ? x->warn != 0 : true;
  S->prof.on = x ? x->profile != 0 : false;
  S->persistent = x ? x->persistent != 0 : true;
  S->resident = x ? x->persistent == 1 : true;
  retain_pool_memory(S->device);
  CK(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&S->aux, cudaStreamNonBlocking));
  S->mem.stream = S->mem.fstream = S->stream;
  if (const char* tr = std::getenv("PFE_TRACE"); tr && tr[0] == '1') {
    S->trace = S->mem.alloc<unsigned long long>(kTraceCap);
    CK(cudaMemsetAsync(S->trace, 0, sizeof(unsigned long long) * kTraceCap, S->stream));
  }
  CK(cudaDeviceGetAttribute(&S->sm, cudaDevAttrMultiProcessorCount, S->device));
  S->d = d;
  S->tab = &pfe_host::table_for(d);
  S->max_grid = S->sm * std::max(8, S->tab->max_blocks_per_sm());
  S->partials = S->mem.alloc<double>(static_cast<size_t>(S->max_grid) * 3 * pfe_dev::kMaxD);
  S->partials_b = S->mem.alloc<double>(static_cast<size_t>(S->max_grid) * pfe_dev::kMaxD);
  S->totals = S->mem.alloc<double>(4 * pfe_dev::kMaxD);
  S->partials_c = S->mem.alloc<double>(static_cast<size_t>(S->sm) * 6 * pfe_dev::kMaxD);
  S->ctl = S->mem.alloc<Ctl>(1);
  CK(cudaMemsetAsync(S->ctl, 0, sizeof(Ctl), S->stream));
  S->h_ctl = static_cast<Ctl*>(pinned_ctl_pool().get(sizeof(Ctl)));
  if (!S->h_ctl) throw Error(PFE_CUDA_ERROR, "cudaMallocHost failed for the control block");
  CK(cudaEventCreate(&S->ev0));
  CK(cudaEventCreate(&S->ev1));
  std::memset(S->h_ctl, 0, sizeof(Ctl));
}

// deg and sqrt(deg) in device row order (after build_topology chose it).
void upload_degree(pfe_solver* S, const double* degree) {
  if (S->deg && S->sqd) return;  // built with the device grid topology
  const int n = S->n;
  std::vector<double> deg(n), sqd(n);
  for (int v = 0; v < n; ++v) {
    const int x = S->perm_h.empty() ? v : S->perm_h[v];
    deg[x] = degree[v];
    sqd[x] = std::sqrt(degree[v]);
  }
  S->deg = S->mem.upload(deg, S->stream);
  S->sqd = S->mem.upload(sqd, S->stream);
}

// TSQR grid: about 8 tiles of rows per block, at most max_grid blocks.
int qr_blocks_for(const pfe_solver* S, long n) {
  const long rows_per_block = 8L * (pfe_dev::kQrRows - S->d);
  return static_cast<int>(std::max<long>(1, std::min<long>((n + rows_per_block - 1) / rows_per_block, S->max_grid)));
}

pfe_solver* create_solver(const pfe_graph* g, const pfe_params* p, const pfe_exec* x) {
  if (!g || !p) config_error("null graph or params");
  const auto t0 = std::chrono::steady_clock::now();
  HostGraph hg{g->n, static_cast<long>(g->m), g->ei, g->ej, g->w, g->degree};
  NvtxRange nv_create("pfe solver create");
  {
    NvtxRange nv("pfe validate");
    validate(hg, *p, true);
  }
  if (g->m > 0x3fffffffL) config_error("graph too large for 32-bit edge indices");
  auto S = std::make_unique<pfe_solver>();
  S->prm = *p;
  // IC(0) (the reference default): general-graph kernels, host-driven PCG
  // loop with the device triangular solves after init and every update
  S->ic = p->preconditioner == PFE_PRECOND_IC0;
  S->jacobi_fallback = false;
  init_common(S.get(), x, p->dim);
  if (S->ic) {
    S->use_graphs = false;
    S->persistent = false;
    S->resident = false;
  }
  S->n = g->n;
  S->m = g->m;
  const auto t1 = std::chrono::steady_clock::now();
  {
    NvtxRange nv("pfe topology");
    build_topology(S.get(), hg, S->ic ? 0 : g->grid_h, S->ic ? 0 : g->grid_w, S->ic ? 0 : g->grid_radius);
  }
  const auto t2 = std::chrono::steady_clock::now();
  upload_degree(S.get(), g->degree);
  S->qr_blocks = qr_blocks_for(S.get(), g->n);
  S->rbuf = S->mem.alloc<double>(static_cast<size_t>(S->qr_blocks) * S->d * S->d);
  S->wmat = S->mem.alloc<double>(static_cast<size_t>(S->d) * S->d);
  S->ensure_log(64);
  CK(cudaStreamSynchronize(S->stream));
  const auto t3 = std::chrono::steady_clock::now();
  S->setup_s = std::chrono::duration<double>(t3 - t0).count();
  if (const char* e = std::getenv("PFE_SETUP_TIMING"); e && e[0] == '1') {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "pfe_solver_create: validate + init %.2f ms, topology %.2f ms, degree + sync %.2f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  return S.release();
}

// ------------------------------------------------------------- state ------

// Column-major host layout <-> device rows (perm: vertex -> device row, or null).
__global__ void k_colmajor_to_rows(long n, int d, const double* __restrict__ src, double* dst,
                                   const int* __restrict__ perm) {
  const long total = n * d, stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long v = e / d;
    const int j = static_cast<int>(e - v * d);
    dst[(perm ? perm[v] : v) * d + j] = src[v + j * n];
  }
}
__global__ void k_rows_to_colmajor(long n, int d, const double* __restrict__ src, double* dst,
                                   const int* __restrict__ perm) {
  const long total = n * d, stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long v = e % n;
    const int j = static_cast<int>(e / n);
    dst[e] = src[(perm ? perm[v] : v) * d + j];
  }
}
__global__ void k_scale_rows(long n, int d, const double* __restrict__ s, const double* __restrict__ y, double* out) {
  const long total = n * d, stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride)
    out[e] = s[e / d] * y[e];
}

// host col-major n x d -> device row-major via a staging buffer
// (ld: distance between the host columns, n when they are contiguous; a row
// band uploads its rows of each column of the global matrix)
void upload_rows(pfe_solver* S, const double* host, long n, int d, double* dst, double* staging, long ld = 0) {
  if (ld == 0 || ld == n) {
    copy_h2d(staging, host, sizeof(double) * n * d, S->stream);
  } else {
    for (int j = 0; j < d; ++j) copy_h2d(staging + j * n, host + j * ld, sizeof(double) * n, S->stream);
  }
  k_colmajor_to_rows<<<S->grid_for(n * d), pfe_dev::kBlock, 0, S->stream>>>(n, d, staging, dst,
                                                                             n == S->n ? S->perm_d : nullptr);
  CK(cudaGetLastError());
}
void download_rows(pfe_solver* S, const double* src, long n, int d, double* host, double* staging) {
  NvtxRange nv("pfe download");
  k_rows_to_colmajor<<<S->grid_for(n * d), pfe_dev::kBlock, 0, S->stream>>>(n, d, src, staging,
                                                                             n == S->n ? S->perm_d : nullptr);
  CK(cudaGetLastError());
  copy_d2h(host, staging, sizeof(double) * n * d, S->stream);
}

void state_init_from_y0(pfe_state* st) {
  pfe_solver* S = st->s;
  const long nd = static_cast<long>(S->n) * S->d;
  CK(cudaMemcpyAsync(st->y, st->y0, sizeof(double) * nd, cudaMemcpyDeviceToDevice, S->stream));
  if (S->sqd) {
    k_scale_rows<<<S->grid_for(nd), pfe_dev::kBlock, 0, S->stream>>>(S->n, S->d, S->sqd, st->y0, st->p);
    CK(cudaGetLastError());
  } else {  // operator-only solvers (pfe_pcg_solve_multi) have no degree vector
    CK(cudaMemsetAsync(st->p, 0, sizeof(double) * nd, S->stream));
  }
  CK(cudaMemsetAsync(st->breg, 0, sizeof(double) * nd, S->stream));
  st->inner_zero = true;
  st->rq_valid = false;
}

pfe_state* create_state(pfe_solver* S, const double* y0_host, long y0_ld = 0) {
  NvtxRange nv("pfe state create");
  auto st = std::make_unique<pfe_state>();
  st->s = S;
  st->device = S->device;
  st->mem.stream = S->stream;
  const size_t nd = static_cast<size_t>(S->n) * S->d;
  const size_t ed = static_cast<size_t>(S->edge_rows) * S->d;
  st->y = st->ybuf[0] = st->mem.alloc<double>(nd);
  st->y2 = st->ybuf[1] = st->mem.alloc<double>(nd);
  st->p = st->mem.alloc<double>(nd);
  st->breg = st->mem.alloc<double>(nd);
  st->rq = st->mem.alloc<double>(nd);
  st->r = st->mem.alloc<double>(nd);
  st->pb[0] = st->mem.alloc<double>(nd);
  st->pb[1] = st->mem.alloc<double>(nd);
  st->q = st->mem.alloc<double>(nd);
  st->y0 = st->mem.alloc<double>(nd);
  st->eb[0] = st->mem.alloc<double>(ed);
  st->eb[1] = st->mem.alloc<double>(ed);
  st->es = st->mem.alloc<double>(ed);
  // absent grid slots must read as exact zeros in every edge array
  CK(cudaMemsetAsync(st->eb[0], 0, sizeof(double) * ed, S->stream));
  CK(cudaMemsetAsync(st->eb[1], 0, sizeof(double) * ed, S->stream));
  CK(cudaMemsetAsync(st->es, 0, sizeof(double) * ed, S->stream));
  upload_rows(S, y0_host, S->n, S->d, st->y0, st->q, y0_ld);
  state_init_from_y0(st.get());
  CK(cudaStreamSynchronize(S->stream));
  return st.release();
}

// ------------------------------------------------------------ drivers -----

void check_flags(pfe_solver* S) {
  S->read_ctl();
  if (S->h_ctl->nonfinite_y) {
    CK(cudaMemsetAsync(&S->ctl->nonfinite_y, 0, sizeof(int), S->stream));
    throw Error(PFE_NUMERICAL_ERROR, "split_bregman: NaN in embedding");
  }
  if (S->h_ctl->deficient) {
    const int def = S->h_ctl->deficient;
    CK(cudaMemsetAsync(&S->ctl->deficient, 0, sizeof(int), S->stream));
    throw Error(PFE_NUMERICAL_ERROR,
                "project_orthogonal: input rank-deficient in " + std::to_string(def) + " column(s)");
  }
}

void warn_from_log(pfe_solver* S, long lo, long hi);

PcgArgs pcg_args(pfe_state* st, const double* rhs) {
  pfe_solver* S = st->s;
  PcgArgs a{};
  a.x0 = st->y;
  a.x = st->y2;
  a.rhs = rhs;
  a.r = st->r;
  a.pbuf[0] = st->pb[0];
  a.pbuf[1] = st->pb[1];
  a.q = st->q;
  a.ctl = S->ctl;
  a.part_a = S->partials;
  a.part_b = S->partials_b;
  a.rd_a = S->partials;
  a.rd_b = S->partials_b;
  a.rank_major = 0;
  S->tab->pcg_grids(S->topo, S->lv(), &a.nb_init, &a.nb_spmv, &a.nb_update);
  // Large general graphs: producers reduce their own partials (last block)
  // and the consumers read the totals (their gather-bound kernels cannot hide
  // an nb^2 consumer-side reduction).  Grids and small systems keep the
  // consumer-side reduction, which overlaps the consumer's first loads and
  // has no serial tail.
  a.tot_a = S->totals;
  a.tot_b = S->totals + 3 * pfe_dev::kMaxD;
  a.totals = S->ic || (S->topo.kind == pfe_host::kTopoCsr && static_cast<long>(S->n) * S->d >= (1L << 22));
  a.zbuf = S->ic ? S->zbuf : nullptr;
  if (a.totals) {
    a.rd_a = a.tot_a;
    a.rd_b = a.tot_b;
    a.nb_init = a.nb_spmv = a.nb_update = 1;
  }
  a.tol = S->prm.pcg_rel_tol;
  a.max_iter = S->prm.pcg_max_iter;
  a.use_cond = 0;
  a.phase = 0;
  return a;
}

void warn_columns(pfe_solver* S) {
  if (!S->warn) return;
  for (int j = 0; j < S->d; ++j) {
    const int stt = S->h_ctl->col[j].status;
    if (stt == pfe_dev::kMaxIter || stt == pfe_dev::kFailed)
      std::fprintf(stderr, "pfe: inner solve column %d stopped at rel residual %g\n", j, S->h_ctl->col[j].rel);
  }
}

// One PCG solve of all d columns, host-driven.  The SpMV of iteration k
// decides whether iteration k-1 finished the solve, so the launch sequence
// is spmv(1) [update(k) spmv(k+1)]...; the first burst is sized from the
// previous solve's iteration count (kernels of a finished solve exit at once).
void pcg_solve_host(pfe_state* st, const double* rhs) {
  pfe_solver* S = st->s;
  PcgArgs a = pcg_args(st, rhs);
  const auto L = S->lv();
  const int maxit = S->prm.pcg_max_iter;
  auto spmv = [&](int k) {
    a.phase = pfe_dev::pcg_phase(k);
    S->prof.begin(1, S->stream);
    S->tab->pcg_spmv(S->topo, a, L);
    S->prof.end(S->stream);
  };
  // IC(0): z = M^-1 r by the device triangular solves, and the r.z total
  // the consumers read (slot 2 after init, slot 1 after an update) replaced
  // by the preconditioned one (pcg.cpp:63-66, 85-88)
  using DSeq = std::make_integer_sequence<int, pfe_dev::kMaxD>;
  auto ic_z = [&](double* z, int slot) {
    if (!S->ic) return;
    S->prof.begin(2, S->stream);  // timed with the update class
    ic_apply_dispatch(S->d, DSeq{}, S->icd, a.r, z, S->stream);
    const int grid = std::min(S->max_grid, std::max(1, (S->n + 255) / 256));
    ic_dot_dispatch(S->d, DSeq{}, S->n, a.r, z, S->partials, S->ctl, a.tot_a + slot * S->d, grid, S->stream);
    CK(cudaGetLastError());
    S->prof.end(S->stream);
  };
  auto update = [&](int k) {
    a.phase = pfe_dev::pcg_phase(k);
    S->prof.begin(2, S->stream);
    S->tab->pcg_update(S->topo, a, L);
    S->prof.end(S->stream);
    ic_z(S->zbuf, 1);
  };
  S->prof.begin(0, S->stream);
  S->tab->pcg_init(S->topo, a, L);
  S->prof.end(S->stream);
  ic_z(a.pbuf[0], 2);  // p = z for the first iteration
  int k = 1;
  spmv(1);
  for (int burst = S->ic ? 1 : std::max(1, S->pred_iters);; burst = 1) {
    for (int b = 1; b < burst && k <= maxit; ++b) {
      update(k);
      spmv(++k);
    }
    S->read_ctl();
    if (!S->h_ctl->any_active || k > maxit) break;
    update(k);
    spmv(++k);
  }
  S->pred_iters = std::max(1, S->h_ctl->iter);
  warn_columns(S);
  S->prof.begin(3, S->stream);
  S->tab->pcg_finalize(S->n, st->y, st->y2, S->ctl, S->le());
  S->prof.end(S->stream);
  ++S->inner_launched;
  std::swap(st->y, st->y2);
}

// The same solve captured into the graph being built on S->stream: init,
// then a WHILE node whose body is {spmv, update}; the kernels set the loop
// condition on the device.
void pcg_solve_captured(pfe_state* st, const double* rhs) {
  pfe_solver* S = st->s;
  PcgArgs a = pcg_args(st, rhs);
  const auto L = S->lv();
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(S->stream, &cs, nullptr, &g, &deps, &nd));
  if (cs != cudaStreamCaptureStatusActive || g == nullptr)
    throw Error(PFE_CUDA_ERROR, "graph capture was invalidated before the PCG loop");
  cudaGraphConditionalHandle h;  // 1 at every graph launch; the deciding SpMV clears it
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  a.cond = h;
  a.use_cond = 1;
  S->tab->pcg_init(S->topo, a, L);
  // iteration 1 peeled (p comes from init, x from x0); the WHILE body then
  // runs iterations 2k and 2k+1 with static buffer parities.
  a.phase = 0;
  S->tab->pcg_spmv(S->topo, a, L);
  S->tab->pcg_update(S->topo, a, L);
  CK(cudaGetLastError());
  CK(cudaStreamGetCaptureInfo(S->stream, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &np));
  CK(cudaStreamUpdateCaptureDependencies(S->stream, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(S->aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  for (int ph : {2, 1}) {
    a.phase = ph;
    S->tab->pcg_spmv(S->topo, a, {L.grid, S->aux, S->sm});
    S->tab->pcg_update(S->topo, a, {L.grid, S->aux, S->sm});
  }
  CK(cudaGetLastError());
  CK(cudaStreamEndCapture(S->aux, &body));
  S->tab->pcg_finalize(S->n, st->y, st->y2, S->ctl, S->le());
  ++S->inner_launched;
  std::swap(st->y, st->y2);
}

struct RunMode {
  bool captured;
  pfe_iterate_fn cb;
  void* user;
};

void solve_step(pfe_state* st, const double* rhs, const RunMode& mode) {
  if (mode.captured)
    pcg_solve_captured(st, rhs);
  else
    pcg_solve_host(st, rhs);
}

// General-graph split-Bregman pass: L2 prefetch of the b_old rows, opt-in
// (PFE_SB_PREFETCH=1).  Measured slower on C5 (1506 -> 1595 us per pass): the
// pass is bound by DRAM throughput on scattered 128-byte rows, not by the
// latency of its gathers, and the prefetches only add L2 requests.
int sb_prefetch() {
  static const int on = [] {
    const char* e = std::getenv("PFE_SB_PREFETCH");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return on;
}

// PfeSolver::split_bregman (solver.cpp:73-108).
void split_bregman_run(pfe_state* st, int max_iter, const RunMode& mode) {
  NvtxRange nv("pfe split_bregman");
  pfe_solver* S = st->s;
  const double hl = 0.5 * S->prm.lambda, hr = 0.5 * S->prm.r, gamma = 1.0 / S->prm.lambda;
  const bool conv = S->prm.conv_tol > 0.0;
  if (!st->rq_valid) {
    S->prof.begin(5, S->stream);
    S->tab->rhs_quad(S->n, S->sqd, st->p, st->breg, st->rq, hr, S->le());
    S->prof.end(S->stream);
    st->rq_valid = true;
  }
  const double* rhs = st->rq;
  if (!st->inner_zero) {
    S->prof.begin(5, S->stream);
    S->tab->rhs_from_state(S->topo, st->es, st->eb[st->eb_cur], st->rq, st->r, hl, S->lv());
    S->prof.end(S->stream);
    rhs = st->r;
  }
  auto after_iteration = [&](int it) -> bool {  // callback + relative-change test; true = stop
    if (mode.cb) {
      std::vector<double> yh(static_cast<size_t>(S->n) * S->d);
      download_rows(S, st->y, S->n, S->d, yh.data(), st->q);
      check_flags(S);
      mode.cb(it, yh.data(), S->n, S->d, mode.user);
    }
    if (conv) {
      S->tab->diff_norms(S->n, st->y, st->y2, S->partials, S->ctl, S->lr());
      S->read_ctl();
      const double den = std::sqrt(S->h_ctl->scalar[2]);
      if (den > 0.0 && std::sqrt(S->h_ctl->scalar[1]) / den <= S->prm.conv_tol) return true;
    }
    return false;
  };
  if (S->persistent && !mode.captured && S->topo.kind != pfe_host::kTopoCsr) {
    // Whole call in one cooperative launch; with a callback or the
    // relative-change test, one launch per inner iteration.
    const bool per_iter = mode.cb != nullptr || conv;
    const long inner_before = S->inner_launched;
    for (int it = 0; it < max_iter;) {
      const int nrun = per_iter ? 1 : max_iter;
      pfe_host::PersistIn in{};
      in.ybuf[0] = st->ybuf[0];
      in.ybuf[1] = st->ybuf[1];
      in.ycur = st->y == st->ybuf[0] ? 0 : 1;
      in.r = st->r;
      in.pbuf[0] = st->pb[0];
      in.pbuf[1] = st->pb[1];
      in.q = st->q;
      in.eb[0] = st->eb[0];
      in.eb[1] = st->eb[1];
      in.ebcur = st->eb_cur;
      in.es = st->es;
      in.rq = st->rq;
      in.rhs0 = rhs;
      in.b_zero = st->inner_zero ? 1 : 0;
      in.n_inner = nrun;
      in.write_s_last = 1;
      in.rhs_last = (it + nrun < max_iter) ? 1 : 0;
      in.tol = S->prm.pcg_rel_tol;
      in.max_iter = S->prm.pcg_max_iter;
      in.hl = hl;
      in.gamma = gamma;
      in.ctl = S->ctl;
      in.part = S->partials;
      in.part_b = S->partials_b;
      in.trace = S->trace;
      in.trace_cap = S->trace ? kTraceCap : 0;
      in.allow_resident = S->resident && S->nranks == 1 ? 1 : 0;
      in.part_c = S->partials_c;
      S->prof.begin(7, S->stream);
      S->persist_kind = S->tab->sb_persistent(S->topo, in, S->lv());
      S->prof.end(S->stream);
      for (int k = 0; k < nrun; ++k) {
        std::swap(st->y, st->y2);
        st->eb_cur ^= 1;
      }
      st->inner_zero = false;
      S->inner_launched += nrun;
      rhs = st->r;
      it += nrun;
      if (per_iter && after_iteration(it - 1)) break;
    }
    // the reference's non-converged-column warnings (solver.cpp:87-92), from
    // the device PCG log of this call's inner iterations
    if (S->warn) warn_from_log(S, inner_before, S->inner_launched);
    return;
  }
  for (int it = 0; it < max_iter; ++it) {
    const bool last = it == max_iter - 1;
    solve_step(st, rhs, mode);
    SbArgs sa{};
    sa.y = st->y;
    sa.b_old = st->inner_zero ? nullptr : st->eb[st->eb_cur];
    sa.b_new = st->eb[st->eb_cur ^ 1];
    sa.s_out = (last || conv || mode.cb) ? st->es : nullptr;
    sa.rq = st->rq;
    sa.rhs = last ? nullptr : st->r;
    sa.hl = hl;
    sa.gamma = gamma;
    sa.ctl = S->ctl;
    sa.prefetch = sb_prefetch();
    S->prof.begin(4, S->stream);
    S->tab->sb_pass(S->topo, sa, S->lv());
    S->prof.end(S->stream);
    st->eb_cur ^= 1;
    st->inner_zero = false;
    rhs = st->r;
    if (after_iteration(it)) break;
  }
}

// Projection + outer Bregman update (solver.cpp:116-118) with the next
// rhs_quad fused into the same pass.
void project_step(pfe_state* st) {
  NvtxRange nv("pfe projection");
  pfe_solver* S = st->s;
  S->prof.begin(6, S->stream);
  S->tab->tsqr_local(S->n, st->y, S->sqd, st->breg, S->rbuf, {S->qr_blocks, S->stream});
  S->tab->tsqr_final(S->qr_blocks, S->rbuf, S->wmat, S->ctl, {1, S->stream});
  S->tab->project_apply(S->n, st->y, S->sqd, st->breg, S->wmat, st->p, st->rq, 0.5 * S->prm.r, S->lr());
  S->prof.end(S->stream);
  st->rq_valid = true;
}

// PfeSolver::run_soc (solver.cpp:110-126).
void run_soc_run(pfe_state* st, int soc_max, int sb_max, const RunMode& mode) {
  pfe_solver* S = st->s;
  const bool conv = S->prm.conv_tol > 0.0;
  const long nd = static_cast<long>(S->n) * S->d;
  if (conv && !st->yout) st->yout = st->mem.alloc<double>(static_cast<size_t>(nd));
  for (int k = 0; k < soc_max; ++k) {
    st->inner_zero = true;
    if (conv) CK(cudaMemcpyAsync(st->yout, st->y, sizeof(double) * nd, cudaMemcpyDeviceToDevice, S->stream));
    split_bregman_run(st, sb_max, mode);
    project_step(st);
    if (!mode.captured) check_flags(S);
    if (conv) {
      S->tab->diff_norms(S->n, st->y, st->yout, S->partials, S->ctl, S->lr());
      S->read_ctl();
      const double den = std::sqrt(S->h_ctl->scalar[2]);
      if (den > 0.0 && std::sqrt(S->h_ctl->scalar[1]) / den <= S->prm.conv_tol) break;
    }
  }
}

// Non-converged-column warnings (solver.cpp:87-92) for iterations run inside a graph.
void warn_from_log(pfe_solver* S, long lo, long hi) {
  hi = std::min(hi, S->log_cap);
  if (hi <= lo) return;
  const size_t k = static_cast<size_t>(hi - lo) * S->d;
  std::vector<int> stt(k);
  std::vector<double> rel(k);
  stream_copy(stt.data(), S->log_st + lo * S->d, sizeof(int) * k, cudaMemcpyDeviceToHost, S->stream);
  stream_copy(rel.data(), S->log_rel + lo * S->d, sizeof(double) * k, cudaMemcpyDeviceToHost, S->stream);
  for (size_t i = 0; i < k; ++i)
    if (stt[i] == pfe_dev::kMaxIter || stt[i] == pfe_dev::kFailed)
      std::fprintf(stderr, "pfe: inner solve column %d stopped at rel residual %g\n", static_cast<int>(i % S->d), rel[i]);
}

enum CallKind { kCallSplit = 0, kCallSoc = 1, kCallTwoStage = 2 };
constexpr int kPieceOuter = 3;  // graph piece: one outer iteration (split_bregman + projection)

// Executes a call either host-driven or as one cached CUDA graph.
void execute_inner(pfe_state* st, int kind, int a0, int a1, pfe_iterate_fn cb, void* user);

// Device time of every call, CUDA events on the solver stream.
void execute(pfe_state* st, int kind, int a0, int a1, pfe_iterate_fn cb, void* user) {
  NvtxRange nv(kind == kCallSplit ? "pfe call split_bregman" : (kind == kCallSoc ? "pfe call run_soc" : "pfe call two_stage"));
  pfe_solver* S = st->s;
  CK(cudaEventRecord(S->ev0, S->stream));
  execute_inner(st, kind, a0, a1, cb, user);
  CK(cudaEventRecord(S->ev1, S->stream));
  CK(cudaEventSynchronize(S->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
  S->last_ms = ms;
}

void execute_inner(pfe_state* st, int kind, int a0, int a1, pfe_iterate_fn cb, void* user) {
  pfe_solver* S = st->s;
  // the persistent path needs no graph (a whole call is ~3 launches per outer step)
  const bool graphable = S->use_graphs && !cb && !(S->prm.conv_tol > 0.0) && !S->prof.on &&
                         !(S->persistent && S->topo.kind != pfe_host::kTopoCsr);
  long planned = 0;
  if (kind == kCallSplit) planned = a0;
  if (kind == kCallSoc) planned = static_cast<long>(a0) * a1;
  if (kind == kCallTwoStage) planned = static_cast<long>(S->prm.soc_max) * S->prm.sb_max_stage1 + std::max(0, S->prm.sb_max_stage2);
  S->ensure_log(planned);
  auto body = [&](const RunMode& mode) {
    if (kind == kCallSplit) {
      split_bregman_run(st, a0, mode);
    } else if (kind == kCallSoc) {
      run_soc_run(st, a0, a1, mode);
    } else {
      run_soc_run(st, S->prm.soc_max, S->prm.sb_max_stage1, mode);
      if (S->prm.sb_max_stage2 > 0) split_bregman_run(st, S->prm.sb_max_stage2, mode);
    }
  };
  if (!graphable) {
    body(RunMode{false, cb, user});
    S->prof.collect();
    check_flags(S);
    return;
  }
  // One cached CUDA graph per (piece, state bookkeeping the capture bakes in).
  // A soc / two_stage call is issued as one graph launch per outer iteration
  // (split_bregman + projection) instead of one graph of the whole call: the
  // graph is soc_max times smaller, which is what a one-call pfe_solve pays to
  // capture, instantiate and destroy (C1: ~15 + 11 ms of a 51 ms call before).
  // With an even sb_max every outer iteration finds the state bookkeeping it
  // started from and relaunches the same executable graph; otherwise two
  // graphs alternate.  The launches are queued back to back; the host waits
  // once, at the end of the call.
  const long first = S->inner_launched;
  auto run_graph = [&](int piece, int g0, auto&& piece_body) {
    const auto key = std::make_tuple(piece, g0, 0, st->y == st->ybuf[0] ? 0 : 1, st->eb_cur, st->inner_zero ? 1 : 0,
                                     st->rq_valid ? 1 : 0);
    auto it = st->graphs.execs.find(key);
    if (it == st->graphs.execs.end()) {
      const Book pre{st->y, st->y2, st->eb_cur, st->inner_zero, st->rq_valid};
      const long inner0 = S->inner_launched;
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(S->stream, cudaStreamCaptureModeRelaxed));
      try {
        piece_body(RunMode{true, nullptr, nullptr});
      } catch (...) {
        cudaStreamEndCapture(S->stream, &graph);
        throw;
      }
      CK(cudaStreamEndCapture(S->stream, &graph));
      GraphEntry ge{};
      CK(cudaGraphInstantiate(&ge.exec, graph, 0));
      CK(cudaGraphDestroy(graph));
      ge.post = Book{st->y, st->y2, st->eb_cur, st->inner_zero, st->rq_valid};
      ge.inner = S->inner_launched - inner0;
      st->y = pre.y;
      st->y2 = pre.y2;
      st->eb_cur = pre.eb_cur;
      st->inner_zero = pre.inner_zero;
      st->rq_valid = pre.rq_valid;
      S->inner_launched = inner0;
      it = st->graphs.execs.emplace(key, ge).first;
    }
    CK(cudaGraphLaunch(it->second.exec, S->stream));
    const GraphEntry& ge = it->second;
    st->y = ge.post.y;
    st->y2 = ge.post.y2;
    st->eb_cur = ge.post.eb_cur;
    st->inner_zero = ge.post.inner_zero;
    st->rq_valid = ge.post.rq_valid;
    S->inner_launched += ge.inner;
  };
  auto outer_steps = [&](int soc_max, int sb_max) {  // run_soc (solver.cpp:110-126), fixed counts
    if (!st->rq_valid) {  // outside the graph, so the first outer iteration shares the others' graph
      S->tab->rhs_quad(S->n, S->sqd, st->p, st->breg, st->rq, 0.5 * S->prm.r, S->le());
      st->rq_valid = true;
    }
    for (int k = 0; k < soc_max; ++k) {
      st->inner_zero = true;
      run_graph(kPieceOuter, sb_max, [&](const RunMode& mode) {
        split_bregman_run(st, sb_max, mode);
        project_step(st);
      });
    }
  };
  if (kind == kCallSplit) {
    run_graph(kCallSplit, a0, [&](const RunMode& mode) { split_bregman_run(st, a0, mode); });
  } else if (kind == kCallSoc) {
    outer_steps(a0, a1);
  } else {
    outer_steps(S->prm.soc_max, S->prm.sb_max_stage1);
    if (S->prm.sb_max_stage2 > 0)
      run_graph(kCallSplit, S->prm.sb_max_stage2,
                [&](const RunMode& mode) { split_bregman_run(st, S->prm.sb_max_stage2, mode); });
  }
  CK(cudaStreamSynchronize(S->stream));
  if (S->warn) warn_from_log(S, first, S->inner_launched);
  check_flags(S);
}

#include "pfe_band.cuh"

}  // namespace

// ================================================================ C ABI ===
extern "C" {

const char* pfe_last_error(void) { return g_last_error.c_str(); }

int64_t pfe_release_cached_memory(int32_t device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return 0;
  }
  DeviceGuard g(device);
  return static_cast<int64_t>(block_cache().flush());
}

pfe_params pfe_params_default(void) {
  pfe_params p{};
  p.dim = 5;
  p.lambda = 100.0;
  p.r = 1.0;
  p.soc_max = 10;
  p.sb_max_stage1 = 5;
  p.sb_max_stage2 = 100;
  p.conv_tol = 1e-4;
  p.pcg_rel_tol = 1e-6;
  p.pcg_max_iter = 1000;
  p.preconditioner = PFE_PRECOND_IC0;
  return p;
}

pfe_exec pfe_exec_default(void) {
  pfe_exec x{};
  x.device = 0;
  x.use_graphs = 1;
  x.warn = 1;
  x.profile = 0;
  x.persistent = 1;
  return x;
}

int pfe_device_check(int32_t device) {
  return guarded([&] { require_device(device); });
}

int pfe_solver_create(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, pfe_solver** out) {
  return guarded([&] { *out = create_solver(g, p, x); });
}

void pfe_solver_destroy(pfe_solver* s) {
  if (!s) return;
  DeviceGuard g(s->device);
  delete s;
}

int pfe_solver_report(const pfe_solver* s, pfe_report* out) {
  return guarded([&] {
    pfe_report r{};
    r.topology = s->topo.kind;
    r.n = s->n;
    r.m = s->m;
    r.d = s->d;
    r.jacobi_fallback = s->jacobi_fallback ? 1 : 0;
    r.persistent_kind = s->persist_kind;
    r.setup_seconds = s->setup_s;
    const long cnt = std::min(s->inner_launched, s->log_cap);
    std::vector<int> it(static_cast<size_t>(cnt) * s->d), stt(static_cast<size_t>(cnt) * s->d);
    if (cnt > 0) {
      stream_copy(it.data(), s->log_it, sizeof(int) * it.size(), cudaMemcpyDeviceToHost, s->stream);
      stream_copy(stt.data(), s->log_st, sizeof(int) * stt.size(), cudaMemcpyDeviceToHost, s->stream);
    }
    r.inner_iterations = cnt;
    for (long i = 0; i < cnt; ++i) {
      int mx = 0;
      for (int j = 0; j < s->d; ++j) {
        const int v = it[static_cast<size_t>(i) * s->d + j], st = stt[static_cast<size_t>(i) * s->d + j];
        mx = std::max(mx, v);
        r.pcg_column_iterations += v;
        if (st == pfe_dev::kMaxIter || st == pfe_dev::kFailed) ++r.nonconverged;
        if (st == pfe_dev::kFailed) ++r.failed;
      }
      r.pcg_iterations += mx;
    }
    *out = r;
  });
}

int64_t pfe_solver_pcg_log(const pfe_solver* s, int32_t* iters, int32_t* status, double* rel, int64_t cap) {
  int64_t cnt = 0;
  const int rc = guarded([&] {
    cnt = std::min<int64_t>(std::min(s->inner_launched, s->log_cap), cap);
    if (cnt <= 0) return;
    const size_t k = static_cast<size_t>(cnt) * s->d;
    if (iters) stream_copy(iters, s->log_it, sizeof(int) * k, cudaMemcpyDeviceToHost, s->stream);
    if (status) stream_copy(status, s->log_st, sizeof(int) * k, cudaMemcpyDeviceToHost, s->stream);
    if (rel) stream_copy(rel, s->log_rel, sizeof(double) * k, cudaMemcpyDeviceToHost, s->stream);
  });
  return rc == PFE_OK ? cnt : -rc;
}

int pfe_solver_kernel_times(const pfe_solver* s, pfe_kernel_times* out, int reset) {
  return guarded([&] {
    auto* S = const_cast<pfe_solver*>(s);
    S->prof.collect();
    for (int i = 0; i < PFE_KERNEL_CLASSES; ++i) {
      out->ms[i] = S->prof.ms[i];
      out->launches[i] = S->prof.cnt[i];
      if (reset) {
        S->prof.ms[i] = 0.0;
        S->prof.cnt[i] = 0;
      }
    }
  });
}

double pfe_solver_last_ms(const pfe_solver* s) { return s ? s->last_ms : -1.0; }

int64_t pfe_solver_trace(const pfe_solver* s, uint64_t* out, int64_t cap) {
  int64_t cnt = 0;
  const int rc = guarded([&] {
    if (!s->trace) return;
    cnt = std::min<int64_t>(cap, kTraceCap);
    stream_copy(out, s->trace, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost, s->stream);
  });
  return rc == PFE_OK ? cnt : -rc;
}

int pfe_state_create(pfe_solver* s, const double* y0, pfe_state** out) {
  return guarded([&] {
    if (!y0) config_error("PfeSolver: initial embedding has wrong shape");
    CK(cudaSetDevice(s->device));
    *out = s->part == 1 ? create_band_state(s, y0) : (s->part == 2 ? create_range_state(s, y0) : create_state(s, y0));
  });
}

int pfe_state_reset(pfe_state* st) {
  return guarded([&] {
    CK(cudaSetDevice(st->s->device));
    state_init_from_y0(st);
  });
}

void pfe_state_destroy(pfe_state* st) {
  if (!st) return;
  DeviceGuard g(st->device);
  delete st;
}

// The edge -> device-row map on the host (state get / set of split_b and
// split_s, edge order), downloaded on first use when the topology was
// built on the device.
const std::vector<long>& host_edge_rows(pfe_solver* S) {
  if (S->edge_row.empty() && S->d_edge_slot && S->m > 0) {
    std::vector<int32_t> t(static_cast<size_t>(S->m));
    stream_copy(t.data(), S->d_edge_slot, sizeof(int32_t) * t.size(), cudaMemcpyDeviceToHost, S->stream);
    S->edge_row.assign(t.begin(), t.end());
  }
  return S->edge_row;
}

int pfe_state_get(pfe_state* st, int32_t field, double* out) {
  return guarded([&] {
    pfe_solver* S = st->s;
    CK(cudaSetDevice(S->device));
    const int d = S->d;
    if (S->part) {  // partitioned solver: the global Y, gathered from every band / range
      if (field != PFE_FIELD_Y) config_error("row-band solvers expose the gathered embedding Y only");
      Team t{{st}, false};
      team_gather_y(t, out);
      return;
    }
    if (field <= PFE_FIELD_BREGMAN) {
      const double* src = field == PFE_FIELD_Y ? st->y : (field == PFE_FIELD_P ? st->p : st->breg);
      download_rows(S, src, S->n, d, out, st->q);
      return;
    }
    if (field != PFE_FIELD_SPLIT_B && field != PFE_FIELD_SPLIT_S) config_error("pfe_state_get: unknown field");
    const long m = S->m;
    if (st->inner_zero) {
      std::fill(out, out + m * d, 0.0);
      return;
    }
    const double* src = field == PFE_FIELD_SPLIT_B ? st->eb[st->eb_cur] : st->es;
    std::vector<double> rows(static_cast<size_t>(S->edge_rows) * d);
    stream_copy(rows.data(), src, sizeof(double) * rows.size(), cudaMemcpyDeviceToHost, S->stream);
    const std::vector<long>& er = host_edge_rows(S);
    for (long e = 0; e < m; ++e)
      for (int j = 0; j < d; ++j) out[e + j * m] = rows[static_cast<size_t>(er[e]) * d + j];
  });
}

int pfe_state_set(pfe_state* st, int32_t field, const double* in) {
  return guarded([&] {
    pfe_solver* S = st->s;
    CK(cudaSetDevice(S->device));
    const int d = S->d;
    if (S->part) config_error("partitioned (multi-GPU) solvers take their state from make_state only");
    if (field <= PFE_FIELD_BREGMAN) {
      double* dst = field == PFE_FIELD_Y ? st->y : (field == PFE_FIELD_P ? st->p : st->breg);
      upload_rows(S, in, S->n, d, dst, st->q);
      CK(cudaStreamSynchronize(S->stream));
      if (field != PFE_FIELD_Y) st->rq_valid = false;
      return;
    }
    if (field != PFE_FIELD_SPLIT_B && field != PFE_FIELD_SPLIT_S) config_error("pfe_state_set: unknown field");
    const long m = S->m;
    // materialize both edge arrays before a partial update of one of them
    std::vector<double> b_rows(static_cast<size_t>(S->edge_rows) * d, 0.0), s_rows(b_rows.size(), 0.0);
    if (!st->inner_zero) {
      stream_copy(b_rows.data(), st->eb[st->eb_cur], sizeof(double) * b_rows.size(), cudaMemcpyDeviceToHost, S->stream);
      stream_copy(s_rows.data(), st->es, sizeof(double) * s_rows.size(), cudaMemcpyDeviceToHost, S->stream);
    }
    std::vector<double>& tgt = field == PFE_FIELD_SPLIT_B ? b_rows : s_rows;
    const std::vector<long>& er = host_edge_rows(S);
    for (long e = 0; e < m; ++e)
      for (int j = 0; j < d; ++j) tgt[static_cast<size_t>(er[e]) * d + j] = in[e + j * m];
    stream_copy(st->eb[st->eb_cur], b_rows.data(), sizeof(double) * b_rows.size(), cudaMemcpyHostToDevice, S->stream);
    stream_copy(st->es, s_rows.data(), sizeof(double) * s_rows.size(), cudaMemcpyHostToDevice, S->stream);
    st->inner_zero = false;
  });
}

int pfe_split_bregman(pfe_solver* s, pfe_state* st, int32_t max_iter, pfe_iterate_fn cb, void* user) {
  return guarded([&] {
    CK(cudaSetDevice(s->device));
    if (max_iter <= 0) return;
    if (s->part) {
      if (cb || s->prm.conv_tol > 0.0) config_error("row-band solvers run fixed iteration counts without callbacks");
      Team t{{st}, false};
      s->ensure_log(max_iter);
      team_split_bregman(t, max_iter);
      team_check(t);
      return;
    }
    execute(st, kCallSplit, max_iter, 0, cb, user);
  });
}

int pfe_run_soc(pfe_solver* s, pfe_state* st, int32_t soc_max, int32_t sb_max) {
  return guarded([&] {
    CK(cudaSetDevice(s->device));
    if (soc_max <= 0) return;
    if (s->part) {
      if (s->prm.conv_tol > 0.0) config_error("row-band solvers run fixed iteration counts (conv_tol = 0)");
      Team t{{st}, false};
      band_timed(s, [&] { team_run_soc(t, soc_max, std::max(0, sb_max)); });
      return;
    }
    execute(st, kCallSoc, soc_max, std::max(0, sb_max), nullptr, nullptr);
  });
}

int pfe_two_stage(pfe_solver* s, pfe_state* st) {
  return guarded([&] {
    CK(cudaSetDevice(s->device));
    if (s->part) {
      if (s->prm.conv_tol > 0.0) config_error("row-band solvers run fixed iteration counts (conv_tol = 0)");
      Team t{{st}, false};
      band_timed(s, [&] {
        team_run_soc(t, s->prm.soc_max, s->prm.sb_max_stage1);
        if (s->prm.sb_max_stage2 > 0) {
          s->ensure_log(s->prm.sb_max_stage2);
          team_split_bregman(t, s->prm.sb_max_stage2);
          team_check(t);
        }
      });
      return;
    }
    execute(st, kCallTwoStage, 0, 0, nullptr, nullptr);
  });
}

int pfe_state_objective(pfe_solver* s, pfe_state* st, double* out) {
  return guarded([&] {
    CK(cudaSetDevice(s->device));
    s->tab->objective(s->topo, st->y, s->partials, s->ctl, s->lv());
    CK(cudaGetLastError());
    s->read_ctl();
    *out = s->h_ctl->scalar[0];
  });
}

int pfe_solve(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int32_t mode, const double* y0,
              double* y_out, pfe_report* rep) {
  return guarded([&] {
    // PFE_E2E_TIMING=1: wall time of each stage on stderr
    static const bool timing = [] {
      const char* e = std::getenv("PFE_E2E_TIMING");
      return e && e[0] == '1';
    }();
    auto now = [] { return std::chrono::steady_clock::now(); };
    NvtxRange nv("pfe_solve");
    auto t0 = now();
    std::unique_ptr<pfe_solver> S(create_solver(g, p, x));
    auto t1 = now();
    std::unique_ptr<pfe_state> st(create_state(S.get(), y0));
    auto t2 = now();
    if (mode == 1)
      execute(st.get(), kCallTwoStage, 0, 0, nullptr, nullptr);
    else
      execute(st.get(), kCallSoc, p->soc_max, p->sb_max_stage1, nullptr, nullptr);
    auto t3 = now();
    download_rows(S.get(), st->y, S->n, S->d, y_out, st->q);
    if (rep && pfe_solver_report(S.get(), rep) != PFE_OK) throw Error(PFE_CUDA_ERROR, g_last_error);
    auto t4 = now();
    st.reset();
    S.reset();
    auto t5 = now();
    if (timing) {
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "pfe_solve: create %.2f state %.2f solve %.2f download+report %.2f destroy %.2f ms\n",
                   ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5));
    }
  });
}

int pfe_split_bregman_standalone(const pfe_graph* g, const double* p, const double* b, const pfe_params* prm,
                                 int32_t d, const double* y_init, int32_t max_iter, const pfe_exec* x,
                                 double* y_out, pfe_iterate_fn cb, void* user) {
  return guarded([&] {
    if (!prm) config_error("null params");
    pfe_params local = *prm;
    local.dim = d;  // solver.cpp:142-143
    HostGraph hg{g->n, static_cast<long>(g->m), g->ei, g->ej, g->w, g->degree};
    validate(hg, local, false);
    auto S = std::make_unique<pfe_solver>();
    S->prm = local;
    S->warn = false;  // the standalone entry point does not warn (solver.cpp:161-180)
    S->ic = local.preconditioner == PFE_PRECOND_IC0;  // solver.cpp:150-151 builds a PcgOperator
    S->jacobi_fallback = false;
    init_common(S.get(), x, d);
    S->warn = false;
    if (S->ic) {
      S->use_graphs = false;
      S->persistent = false;
      S->resident = false;
    }
    S->n = g->n;
    S->m = g->m;
    build_topology(S.get(), hg, S->ic ? 0 : g->grid_h, S->ic ? 0 : g->grid_w, S->ic ? 0 : g->grid_radius);
    upload_degree(S.get(), g->degree);
    S->qr_blocks = 1;
    S->rbuf = S->mem.alloc<double>(static_cast<size_t>(d) * d);
    S->wmat = S->mem.alloc<double>(static_cast<size_t>(d) * d);
    std::unique_ptr<pfe_state> st(create_state(S.get(), y_init));
    upload_rows(S.get(), p, S->n, d, st->p, st->q);
    upload_rows(S.get(), b, S->n, d, st->breg, st->q);
    st->rq_valid = false;
    if (max_iter > 0) execute(st.get(), kCallSplit, max_iter, 0, cb, user);
    download_rows(S.get(), st->y, S->n, d, y_out, st->q);
  });
}

int pfe_pcg_solve_multi(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* values, int32_t d,
                        const double* b, const double* x0, double rel_tol, int32_t max_iter, int32_t preconditioner,
                        const pfe_exec* x, double* x_out, int32_t* iterations, int32_t* converged, double* residual,
                        int32_t* jacobi_fallback) {
  return guarded([&] {
    if (rel_tol <= 0.0) config_error("PcgOperator: rel_tol must be > 0");
    if (max_iter < 1) config_error("PcgOperator: max_iter must be >= 1");
    if (n < 1 || d < 1 || d > pfe_dev::kMaxD) config_error("pcg_solve_multi: dimension mismatch");
    auto S = std::make_unique<pfe_solver>();
    S->prm = pfe_params_default();
    S->prm.dim = d;
    S->prm.pcg_rel_tol = rel_tol;
    S->prm.pcg_max_iter = max_iter;
    S->prm.preconditioner = preconditioner;
    S->warn = false;
    init_common(S.get(), x, d);
    S->warn = false;
    S->n = n;
    S->m = 0;
    const int nnz = row_ptr[n];
    std::vector<int> aptr(row_ptr, row_ptr + n + 1), acol(col_idx, col_idx + nnz);
    std::vector<double> aval(values, values + nnz), invd(n, 1.0);
    if (preconditioner != PFE_PRECOND_NONE)
      for (int r = 0; r < n; ++r)
        for (int k = aptr[r]; k < aptr[r + 1]; ++k)
          if (acol[k] == r && aval[k] > 0.0) invd[r] = 1.0 / aval[k];  // pcg.cpp:15-20
    pfe_dev::Csr c{};
    c.n = n;
    c.vb = 0;
    c.ve = n;
    c.aptr = S->mem.upload(aptr, S->stream);
    c.acol = S->mem.upload(acol, S->stream);
    c.aval = S->mem.upload(aval, S->stream);
    c.invd = S->mem.upload(invd, S->stream);
    S->topo.kind = pfe_host::kTopoCsr;
    S->topo.csr = c;
    S->edge_rows = 0;
    if (preconditioner == PFE_PRECOND_IC0) {  // PcgOperator ctor, pcg.cpp:22-28
      S->ic = true;
      std::vector<int> ident(static_cast<size_t>(n));
      std::iota(ident.begin(), ident.end(), 0);
      build_ic(S.get(), n, aptr, acol, aval, ident);  // breakdown: Jacobi + jacobi_fallback
    }
    std::unique_ptr<pfe_state> st(create_state(S.get(), x0));
    upload_rows(S.get(), b, n, d, st->r, st->q);
    S->ensure_log(1);
    pcg_solve_host(st.get(), st->r);
    download_rows(S.get(), st->y, n, d, x_out, st->q);
    S->read_ctl();
    for (int j = 0; j < d; ++j) {
      const auto& col = S->h_ctl->col[j];
      const bool ok = col.status == pfe_dev::kConverged || col.status == pfe_dev::kConvInit ||
                      col.status == pfe_dev::kZeroRhs;
      if (iterations) iterations[j] = col.iters;
      if (converged) converged[j] = ok ? 1 : 0;
      if (residual) residual[j] = col.rel;
      if (jacobi_fallback) jacobi_fallback[j] = S->jacobi_fallback ? 1 : 0;
    }
  });
}

int pfe_ic0_probe(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* values,
                  int32_t* jacobi_fallback) {
  return guarded([&] {
    if (n < 0 || !row_ptr || !jacobi_fallback) config_error("pfe_ic0_probe: bad arguments");
    pfe_host::IcFactorHost f;
    *jacobi_fallback = pfe_host::ic0_factor(n, row_ptr, col_idx, values, f) ? 0 : 1;
  });
}

int pfe_objective(const pfe_graph* g, int32_t d, const double* y, const pfe_exec* x, double* out) {
  return guarded([&] {
    pfe_params p = pfe_params_default();
    p.dim = d;
    p.lambda = 2.0;  // operator unused; any valid values
    std::vector<double> unit;
    pfe_graph gg = *g;
    if (!gg.degree) {
      unit.assign(g->n, 1.0);
      gg.degree = unit.data();
    }
    HostGraph hg{gg.n, static_cast<long>(gg.m), gg.ei, gg.ej, gg.w, gg.degree};
    if (gg.n < 1) config_error("objective: dimension mismatch");
    for (long k = 0; k < hg.m; ++k) {
      if (hg.ei[k] < 0 || hg.ei[k] >= hg.n || hg.ej[k] < 0 || hg.ej[k] >= hg.n || hg.ei[k] >= hg.ej[k])
        config_error("objective: invalid edge " + std::to_string(k));
    }
    auto S = std::make_unique<pfe_solver>();
    S->prm = p;
    init_common(S.get(), x, d);
    S->n = gg.n;
    S->m = gg.m;
    build_topology(S.get(), hg, gg.grid_h, gg.grid_w, gg.grid_radius);
    double* dy = S->mem.alloc<double>(static_cast<size_t>(gg.n) * d);
    double* stg = S->mem.alloc<double>(static_cast<size_t>(gg.n) * d);
    upload_rows(S.get(), y, gg.n, d, dy, stg);
    S->tab->objective(S->topo, dy, S->partials, S->ctl, S->lv());
    CK(cudaGetLastError());
    S->read_ctl();
    *out = S->h_ctl->scalar[0];
  });
}

}  // extern "C"

__global__ void k_shrink(long count, const double* __restrict__ v, double gamma, double* out) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += stride)
    out[e] = pfe_dev::shrink1(v[e], gamma);
}

extern "C" {

int pfe_shrink(int64_t count, const double* v, double gamma, const pfe_exec* x, double* out) {
  return guarded([&] {
    if (gamma < 0.0) config_error("shrink: gamma must be >= 0");
    require_device(x ? x->device : 0);
    if (count <= 0) return;
    double *dv = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dv, sizeof(double) * count));
    CK(cudaMalloc(&dout, sizeof(double) * count));
    CK(cudaMemcpy(dv, v, sizeof(double) * count, cudaMemcpyHostToDevice));
    k_shrink<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 4096)), 256>>>(count, dv, gamma, dout);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost);
    cudaFree(dv);
    cudaFree(dout);
    CK(e);
  });
}

int pfe_band_plan(int32_t height, int32_t nranks, int32_t radius, int32_t rank, int32_t* out) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks || radius < 0) config_error("pfe_band_plan: bad arguments");
    const BandPlan bp = band_plan(height, nranks, radius, rank);
    out[0] = bp.r0;
    out[1] = bp.r1;
    out[2] = bp.lo;
    out[3] = bp.hi;
  });
}

int pfe_nccl_unique_id(uint8_t* out) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == PFE_NCCL_ID_BYTES, "NCCL unique id size");
    std::memcpy(out, &id, sizeof(id));
  });
}

int pfe_solver_create_band(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, const uint8_t* nccl_id,
                           int32_t nranks, int32_t rank, pfe_solver** out) {
  return guarded([&] {
    require_device(x ? x->device : 0);
    // (a one-rank team gets a communicator too: its gathers run through NCCL
    // like any other team's, which is how the one-GPU test box exercises the
    // process-per-GPU path)
    if (!nccl_id) config_error("pfe_solver_create_band: null NCCL id");
    ncclComm_t comm = nullptr;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    nccl_check(nccl().CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    try {
      *out = g && g->grid_h > 0 ? create_band_solver(g, p, x, nranks, rank, comm)
                                : create_range_solver(g, p, x, nranks, rank, comm);
    } catch (...) {
      if (comm) nccl().CommDestroy(comm);
      throw;
    }
  });
}

int pfe_range_partition_stats(const pfe_graph* g, int32_t nranks, int64_t* owned, int64_t* ghosts, int64_t* sends) {
  return guarded([&] { range_partition_stats(g, nranks, owned, ghosts, sends); });
}

int pfe_solve_banded(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int32_t nbands, int32_t mode,
                     const double* y0, double* y_out, pfe_report* rep) {
  return guarded([&] {
    std::vector<std::unique_ptr<pfe_solver>> solvers;
    std::vector<std::unique_ptr<pfe_state>> states;
    Team t;
    t.emulated = true;
    for (int b = 0; b < nbands; ++b) {
      const bool grid = g && g->grid_h > 0;
      solvers.emplace_back(grid ? create_band_solver(g, p, x, nbands, b, nullptr)
                                : create_range_solver(g, p, x, nbands, b, nullptr));
      states.emplace_back(grid ? create_band_state(solvers.back().get(), y0)
                               : create_range_state(solvers.back().get(), y0));
      t.st.push_back(states.back().get());
    }
    team_run_soc(t, p->soc_max, p->sb_max_stage1);
    if (mode == 1 && p->sb_max_stage2 > 0) {
      for (auto& s : solvers) s->ensure_log(p->sb_max_stage2);
      team_split_bregman(t, p->sb_max_stage2);
      team_check(t);
    }
    team_gather_y(t, y_out);
    if (rep && pfe_solver_report(solvers[0].get(), rep) != PFE_OK) throw Error(PFE_CUDA_ERROR, g_last_error);
  });
}

int pfe_solve_multi_gpu(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int32_t ndev,
                        const int32_t* devices, int32_t mode, const double* y0, double* y_out, pfe_report* rep,
                        double* device_ms) {
  return guarded([&] {
    if (!g || !p) config_error("null graph or params");
    if (ndev < 1 || !devices) config_error("pfe_solve_multi_gpu: need at least one device");
    std::vector<int> devs(devices, devices + ndev);
    {
      std::vector<int> u = devs;
      std::sort(u.begin(), u.end());
      if (std::adjacent_find(u.begin(), u.end()) != u.end())
        config_error("pfe_solve_multi_gpu: devices must be distinct (pfe_solve_banded emulates bands on one device)");
    }
    for (int dv : devs) require_device(dv);
    // PFE_E2E_TIMING=1: wall time of each stage on stderr
    const bool timing = std::getenv("PFE_E2E_TIMING") && std::getenv("PFE_E2E_TIMING")[0] == '1';
    auto tprev = std::chrono::steady_clock::now();
    auto stage = [&](const char* what) {
      if (!timing) return;
      const auto tn = std::chrono::steady_clock::now();
      std::fprintf(stderr, "pfe_solve_multi_gpu: %-14s %.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(tn - tprev).count());
      tprev = tn;
    };
    // communicators are kept per device list for the life of the process:
    // ncclCommInitAll + destroy cost 0.1-0.5 s per call
    static std::mutex comm_mu;
    static std::map<std::vector<int>, std::vector<ncclComm_t>> comm_cache;
    std::unique_lock<std::mutex> comm_lock(comm_mu);  // one multi-GPU call at a time per process
    auto cit = comm_cache.find(devs);
    if (cit == comm_cache.end()) {
      std::vector<ncclComm_t> fresh(ndev, nullptr);
      nccl_check(nccl().CommInitAll(fresh.data(), ndev, devs.data()), "ncclCommInitAll");
      cit = comm_cache.emplace(devs, fresh).first;
    }
    const std::vector<ncclComm_t>& comms = cit->second;
    stage("ncclCommInitAll");
    const bool grid = g->grid_h > 0;
    std::vector<pfe_solver*> solvers(ndev, nullptr);
    std::vector<pfe_state*> states(ndev, nullptr);
    auto cleanup = [&]() {
      for (int b = 0; b < ndev; ++b) {
        if (states[b]) {
          cudaSetDevice(states[b]->device);
          delete states[b];
        }
        if (solvers[b]) {
          cudaSetDevice(solvers[b]->device);
          solvers[b]->comm = nullptr;  // cached, not owned
          delete solvers[b];
        }
      }
    };
    try {
      Team t;
      {
        // every band's solver and state are built on their own host thread
        // (their set-up is per-device work plus host loops over the band's
        // part of the graph), so the set-up time of a call does not grow with
        // the number of GPUs
        nccl();  // loaded before the threads start
        std::vector<std::exception_ptr> errs(ndev);
        std::vector<std::thread> workers;
        for (int b = 0; b < ndev; ++b)
          workers.emplace_back([&, b] {
            try {
              pfe_exec xb = x ? *x : pfe_exec_default();
              xb.device = devs[b];
              solvers[b] = grid ? create_band_solver(g, p, &xb, ndev, b, comms[b])
                                : create_range_solver(g, p, &xb, ndev, b, comms[b]);
              states[b] = grid ? create_band_state(solvers[b], y0) : create_range_state(solvers[b], y0);
            } catch (...) {
              errs[b] = std::current_exception();
            }
          });
        for (auto& w : workers) w.join();
        for (int b = 0; b < ndev; ++b)
          if (errs[b]) std::rethrow_exception(errs[b]);
        for (int b = 0; b < ndev; ++b) t.st.push_back(states[b]);
        stage("create solvers + states");
      }
      for (auto* S : solvers) CK(cudaEventRecord(on(S)->ev0, S->stream));
      team_run_soc(t, p->soc_max, p->sb_max_stage1);
      if (mode == 1 && p->sb_max_stage2 > 0) {
        for (auto* S : solvers) S->ensure_log(p->sb_max_stage2);
        team_split_bregman(t, p->sb_max_stage2);
        team_check(t);
      }
      double worst = 0.0;
      for (auto* S : solvers) {
        CK(cudaEventRecord(on(S)->ev1, S->stream));
        CK(cudaEventSynchronize(S->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
        worst = std::max(worst, static_cast<double>(ms));
      }
      for (auto* S : solvers) S->last_ms = worst;  // device time, max over the GPUs
      if (device_ms) *device_ms = worst;
      stage("solve");
      team_gather_y(t, y_out);
      stage("gather Y");
      if (rep && pfe_solver_report(solvers[0], rep) != PFE_OK) throw Error(PFE_CUDA_ERROR, g_last_error);
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    stage("destroy");
  });
}

int pfe_project_orthogonal(int32_t n, int32_t d, const double* a, const pfe_exec* x, double* p_out) {
  return guarded([&] {
    if (n < d) config_error("project_orthogonal: need rows >= cols");
    if (d < 1 || d > pfe_dev::kMaxD) config_error("project_orthogonal: the B200 kernels support 1 <= cols <= 16");
    auto S = std::make_unique<pfe_solver>();
    init_common(S.get(), x, d);
    S->n = n;
    const int blocks = qr_blocks_for(S.get(), n);
    double* da = S->mem.alloc<double>(static_cast<size_t>(n) * d);
    double* stg = S->mem.alloc<double>(static_cast<size_t>(n) * d);
    double* dp = S->mem.alloc<double>(static_cast<size_t>(n) * d);
    double* rb = S->mem.alloc<double>(static_cast<size_t>(blocks) * d * d);
    double* w = S->mem.alloc<double>(static_cast<size_t>(d) * d);
    upload_rows(S.get(), a, n, d, da, stg);
    S->tab->tsqr_local(n, da, nullptr, nullptr, rb, {blocks, S->stream});
    S->tab->tsqr_final(blocks, rb, w, S->ctl, {1, S->stream});
    S->tab->project_apply(n, da, nullptr, nullptr, w, dp, nullptr, 0.0, S->lr());
    CK(cudaGetLastError());
    check_flags(S.get());
    download_rows(S.get(), dp, n, d, p_out, stg);
  });
}

int pfe_d_orthonormalize(int32_t n, int32_t d, const double* a, const double* degree, double* out) {
  return guarded([&] { pfe_host::d_orthonormalize(n, d, a, degree, out); });
}

int pfe_random_embedding(int32_t n, int32_t d, uint64_t seed, const double* degree, double* out) {
  return guarded([&] { pfe_host::random_embedding(n, d, seed, degree, out); });
}

int pfe_kmeans(int32_t n, int32_t d, const double* points, int32_t k, uint64_t seed, int32_t max_iter,
               int32_t* labels) {
  return guarded([&] { pfe_host::kmeans(n, d, points, k, seed, max_iter, labels); });
}

int pfe_kmeans_device(int32_t n, int32_t d, const double* points, int32_t k, uint64_t seed, int32_t max_iter,
                      int32_t device, int32_t* labels) {
  return guarded([&] {
    require_device(device);
    pfe_host::kmeans_device(n, d, points, k, seed, max_iter, labels);
  });
}

int pfe_gmm_init_device(int32_t n, const double* features, int32_t k, uint64_t seed, const double* degree,
                        int32_t device, double* y_out, double* means_out, double* vars_out, double* weights_out) {
  return guarded([&] {
    require_device(device);
    pfe_host::gmm_init_device(n, features, k, seed, degree, y_out, means_out, vars_out, weights_out);
  });
}

int pfe_knn_graph(int32_t n, int32_t dim, const double* points, int32_t k, int32_t device, int32_t* ei, int32_t* ej,
                  double* w, double* degree, int64_t* m_out, double* sigma_out) {
  return guarded([&] {
    if (!points || !ei || !ej || !w || !degree || !m_out || !sigma_out) config_error("knn_graph: null argument");
    require_device(device);
    const size_t nk = static_cast<size_t>(n) * std::max(k, 0);
    std::vector<double> d2(nk);
    std::vector<int32_t> idx(nk);
    pfe_host::knn_search(n, dim, points, k, d2.data(), idx.data());
    *m_out = pfe_host::knn_graph_from_lists(n, k, d2.data(), idx.data(), ei, ej, w, degree, sigma_out);
  });
}

int pfe_grid_graph(int32_t height, int32_t width, const double* rgb, double sigma_rgb, int32_t radius,
                   double sigma_xy, int32_t device, int32_t* ei, int32_t* ej, double* w, double* degree,
                   int64_t* m_out) {
  return guarded([&] {
    if (!rgb || !ei || !ej || !w || !degree || !m_out) config_error("grid_graph: null argument");
    require_device(device);
    *m_out = pfe_host::grid_graph_device(height, width, rgb, sigma_rgb, radius, sigma_xy, ei, ej, w, degree);
  });
}

}  // extern "C"

namespace pfe_host {
const LaunchTable& table_for(int d) {
  static const LaunchTable tables[16] = {
      make_table<1>(),  make_table<2>(),  make_table<3>(),  make_table<4>(),  make_table<5>(),  make_table<6>(),
      make_table<7>(),  make_table<8>(),  make_table<9>(),  make_table<10>(), make_table<11>(), make_table<12>(),
      make_table<13>(), make_table<14>(), make_table<15>(), make_table<16>()};
  if (d < 1 || d > 16) throw Error(PFE_CONFIG_ERROR, "embedding dimension must be in [1, 16]");
  return tables[d - 1];
}
}  // namespace pfe_host
