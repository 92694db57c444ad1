// Inter-stage transport: receiver mailboxes with epoch flags (CUDA IPC
// exportable), sender outboxes (DIRECT peer stores / P2P copy kernel / HOST
// delegated path), the latency gate thread (injected c_i, R16) and the
// delegate thread of the host path.
//
// Synchronisation: epoch flags in pinned, device-mapped host memory; GPU
// producers post them with a one-thread release-store signal kernel
// (csrc/comm/flags.cu), the gate / delegate threads from the host; each
// stage's host thread polls them before launching the consuming op.
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/adaptra.h"
#include "../kernels/kernels.h"
#include "../util.h"
#include "transport.h"

namespace adaptra {

// One stream per device for gate-issued flag writes: it never waits on
// anything, so it cannot be held behind a blocked stream wait.
cudaStream_t signal_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t st[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (!st[dev]) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaStreamCreateWithPriority(&st[dev], cudaStreamNonBlocking, -1);
    cudaSetDevice(cur);
  }
  return st[dev];
}

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// ------------------------------------------------------------ gate thread
// Pending items wait for their CUDA event; on completion (observed at t) the
// action runs at t + delay.  Actions only launch a signal kernel on the
// device's signal stream (which never waits) or store a host flag.
struct GateItem {
  cudaEvent_t ev;
  int64_t delay;
  std::function<void(int64_t /*ready_t*/, int64_t /*release_t*/)> action;
  int64_t ready_t = -1;
};

class Gate {
 public:
  static Gate& get() {
    static Gate g;
    return g;
  }
  void push(GateItem it) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      waiting_.push_back(std::move(it));
    }
    cv_.notify_one();
  }

 private:
  struct Cmp {
    bool operator()(const GateItem& a, const GateItem& b) const { return a.ready_t + a.delay > b.ready_t + b.delay; }
  };
  Gate() { th_ = std::thread([this] { loop(); }); }
  ~Gate() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_one();
    if (th_.joinable()) th_.join();
  }
  void loop() {
    std::vector<GateItem> local;
    std::priority_queue<GateItem, std::vector<GateItem>, Cmp> timers;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        if (waiting_.empty() && local.empty() && timers.empty()) {
          cv_.wait(lk, [&] { return stop_ || !waiting_.empty(); });
        }
        if (stop_) return;
        while (!waiting_.empty()) {
          local.push_back(std::move(waiting_.front()));
          waiting_.pop_front();
        }
      }
      // poll events in FIFO order (messages of one outbox complete in order)
      for (size_t k = 0; k < local.size();) {
        cudaError_t q = cudaEventQuery(local[k].ev);
        if (q == cudaSuccess) {
          local[k].ready_t = now_ns();
          timers.push(std::move(local[k]));
          local.erase(local.begin() + k);
        } else {
          if (q != cudaErrorNotReady) cudaGetLastError();
          ++k;
        }
      }
      int64_t t = now_ns();
      while (!timers.empty() && timers.top().ready_t + timers.top().delay <= t) {
        GateItem it = timers.top();
        timers.pop();
        it.action(it.ready_t, t);
        t = now_ns();
      }
      if (!local.empty() || !timers.empty()) {
        int64_t wait = 20000;
        if (!timers.empty()) wait = std::min<int64_t>(wait, timers.top().ready_t + timers.top().delay - now_ns());
        if (wait > 2000) std::this_thread::sleep_for(std::chrono::nanoseconds(wait > 50000 ? 50000 : 1000));
        else std::this_thread::yield();
      }
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<GateItem> waiting_;
  bool stop_ = false;
  std::thread th_;
};

// ------------------------------------------------------------ host ring (shm)
struct HostRing {
  std::string name;
  void* base = nullptr;
  size_t size = 0;
  bool owner = false;
  bool registered = false;
  char* data(int64_t bytes, int mb) const { return (char*)base + (size_t)mb * bytes; }
  volatile uint32_t* flags(int64_t bytes, int n_mb) const { return (volatile uint32_t*)((char*)base + (size_t)n_mb * bytes); }
};

static int ring_open(HostRing& r, const char* name, int n_mb, int64_t bytes, bool create) {
  r.name = name;
  r.size = (size_t)n_mb * bytes + (size_t)n_mb * 4 + 4096;
  int fd = shm_open(name, create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) return set_error(ADAPTRA_ELINK, std::string("shm_open failed: ") + name);
  if (create && ftruncate(fd, (off_t)r.size) != 0) {
    close(fd);
    return set_error(ADAPTRA_ELINK, "ftruncate failed");
  }
  r.base = mmap(nullptr, r.size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (r.base == MAP_FAILED) {
    r.base = nullptr;
    return set_error(ADAPTRA_ELINK, "mmap failed");
  }
  r.owner = create;
  if (create) memset(r.base, 0, r.size);
  cudaError_t e = cudaHostRegister(r.base, r.size, cudaHostRegisterPortable);
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  r.registered = true;
  return ADAPTRA_OK;
}

static void ring_close(HostRing& r) {
  if (!r.base) return;
  if (r.registered) cudaHostUnregister(r.base);
  munmap(r.base, r.size);
  if (r.owner) shm_unlink(r.name.c_str());
  r.base = nullptr;
}

// ------------------------------------------------------------ flags (shm)
// Message flags live in pinned, device-mapped host memory (a POSIX shm
// segment, so other processes can map it): producers' GPUs post them with a
// system-scope release store (signal kernel), the gate thread and the delegate
// path post them from the host, and each stage's host thread polls them before
// launching the consuming op (the paper's busy wait).  No GPU
// stream ever waits on another stream's signal, so no hardware-queue or
// co-residency deadlock is possible.
struct FlagShm {
  std::string name;
  volatile uint32_t* h = nullptr;  // host view
  uint32_t* d = nullptr;           // device view (this process)
  size_t size = 0;
  bool owner = false;
};

static std::atomic<int> g_flag_seq{0};

static int flags_open(FlagShm& f, const std::string& name, int n, bool create) {
  f.name = name;
  f.size = ((size_t)n * 4 + 4095) & ~(size_t)4095;
  int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) return set_error(ADAPTRA_ELINK, "shm_open (flags) failed: " + name);
  if (create && ftruncate(fd, (off_t)f.size) != 0) {
    close(fd);
    return set_error(ADAPTRA_ELINK, "ftruncate (flags) failed");
  }
  void* p = mmap(nullptr, f.size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return set_error(ADAPTRA_ELINK, "mmap (flags) failed");
  if (create) memset(p, 0, f.size);
  cudaError_t e = cudaHostRegister(p, f.size, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    munmap(p, f.size);
    return set_error(ADAPTRA_ECUDA, std::string("cudaHostRegister (flags): ") + cudaGetErrorString(e));
  }
  void* dp = nullptr;
  e = cudaHostGetDevicePointer(&dp, p, 0);
  if (e != cudaSuccess) {
    cudaHostUnregister(p);
    munmap(p, f.size);
    return set_error(ADAPTRA_ECUDA, std::string("cudaHostGetDevicePointer: ") + cudaGetErrorString(e));
  }
  f.h = (volatile uint32_t*)p;
  f.d = (uint32_t*)dp;
  f.owner = create;
  return ADAPTRA_OK;
}

static void flags_close(FlagShm& f) {
  if (!f.h) return;
  cudaHostUnregister((void*)f.h);
  munmap((void*)f.h, f.size);
  if (f.owner) shm_unlink(f.name.c_str());
  f.h = nullptr;
}

}  // namespace adaptra

using namespace adaptra;

struct adaptra_inbox {
  int dev = 0, n_mb = 0;
  int64_t bytes = 0;
  void* mbox = nullptr;
  FlagShm fl;                         // uint32[n_mb] epoch flags (host memory, device-mapped)
  HostRing ring;
  bool has_ring = false;
  std::atomic<int> host_on{0};
  cudaStream_t dstream = nullptr;     // delegate H2D stream
  bool own_dstream = false;           // dstream created for this inbox (multi-queue)
  std::vector<uint32_t> delivered;    // host path: epoch delivered per mb
};

struct adaptra_outbox {
  int dev = 0, n_mb = 0, mode = ADAPTRA_LINK_DIRECT;
  int64_t bytes = 0;
  char* peer_mbox = nullptr;
  volatile uint32_t* peer_hflags = nullptr;  // receiver's flags, host view
  uint32_t* peer_dflags = nullptr;           // receiver's flags, this device's view
  FlagShm fl_map;                            // cross-process mapping of the flags
  bool ipc = false;
  void* staging = nullptr;
  HostRing ring;
  bool has_ring = false;
  cudaStream_t lstream = nullptr;  // data movement (P2P copy kernel / D2H)
  std::vector<cudaEvent_t> ev_prod, ev_moved;
  std::atomic<int64_t> latency{0};
  std::atomic<int64_t> n_msgs{0}, sum_delay{0}, max_delay{0};
  std::atomic<int64_t> inflight{0};  // gate items not yet released
  std::atomic<int> force_host{0};    // delegated path by policy (straggler), link still up
  // DIRECT to a mailbox on another GPU: the producer's epilogue writes a local
  // staging slot (TMA stores) and the copy engine moves it over NVLink.  An
  // epilogue storing straight into peer memory ran the FC2 GEMM 1.75x slower
  // and put 4.5x the payload on NVLink (32 B granules;
  // profiles/r02_direct_nvlink.txt).  $ADAPTRA_DIRECT_REMOTE_STORES=1 restores it.
  bool remote_ce = false;
};

static bool remote_stores_forced() {
  static const bool v = getenv("ADAPTRA_DIRECT_REMOTE_STORES") && atoi(getenv("ADAPTRA_DIRECT_REMOTE_STORES")) == 1;
  return v;
}

// ------------------------------------------------------------ delegate thread
namespace adaptra {
class Delegate {
 public:
  static Delegate& get() {
    static Delegate d;
    return d;
  }
  void add(adaptra_inbox* ib) {
    std::lock_guard<std::mutex> lk(mu_);
    boxes_.push_back(ib);
    cv_.notify_one();
  }
  void remove(adaptra_inbox* ib) {
    std::lock_guard<std::mutex> lk(mu_);
    for (size_t k = 0; k < boxes_.size(); ++k)
      if (boxes_[k] == ib) {
        boxes_.erase(boxes_.begin() + k);
        break;
      }
  }

 private:
  Delegate() { th_ = std::thread([this] { loop(); }); }
  ~Delegate() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_one();
    if (th_.joinable()) th_.join();
  }
  void loop() {
    for (;;) {
      bool any = false;
      {
        std::unique_lock<std::mutex> lk(mu_);
        if (stop_) return;
        for (adaptra_inbox* ib : boxes_) {
          if (!ib->host_on.load()) continue;
          any = true;
          volatile uint32_t* hf = ib->ring.flags(ib->bytes, ib->n_mb);
          for (int mb = 0; mb < ib->n_mb; ++mb) {
            uint32_t v = hf[mb];
            if (v > ib->delivered[mb]) {
              // eager receive: H2D into the mailbox on the delegate stream, then the device flag
              cudaSetDevice(ib->dev);
              cudaMemcpyAsync((char*)ib->mbox + (size_t)mb * ib->bytes, ib->ring.data(ib->bytes, mb), ib->bytes,
                              cudaMemcpyHostToDevice, ib->dstream);
              stream_write(ib->dstream, ib->fl.d + mb, v);
              ib->delivered[mb] = v;
            }
          }
        }
        if (!any) cv_.wait_for(lk, std::chrono::milliseconds(5));
      }
      if (any) std::this_thread::sleep_for(std::chrono::microseconds(2));
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<adaptra_inbox*> boxes_;
  bool stop_ = false;
  std::thread th_;
};
}  // namespace adaptra

// ================================================================ inbox
extern "C" int adaptra_inbox_create(int32_t dev, int32_t n_mb, int64_t bytes, const char* host_name,
                                    adaptra_inbox_t* out) {
  if (n_mb < 1 || bytes < 16 || bytes % 16 || !out) return set_error(ADAPTRA_EINVAL, "inbox_create: bad args");
  auto* ib = new adaptra_inbox();
  ib->dev = dev;
  ib->n_mb = n_mb;
  ib->bytes = bytes;
  ib->delivered.assign(n_mb, 0);
  cudaSetDevice(dev);
  if (cudaMalloc(&ib->mbox, (size_t)n_mb * bytes) != cudaSuccess) {
    delete ib;
    return set_error(ADAPTRA_ENOMEM, "inbox_create: cudaMalloc failed");
  }
  {
    const std::string nm = "/adaptra_fl_" + std::to_string((long)getpid()) + "_" + std::to_string(g_flag_seq++);
    int rc = flags_open(ib->fl, nm, n_mb, true);
    if (rc) {
      cudaFree(ib->mbox);
      delete ib;
      return rc;
    }
  }
  // Multi-queue delegated path: every inbox (one
  // link direction) gets its own H2D stream, so host-path deliveries of
  // different links proceed on separate copy queues instead of one.
  // ADAPTRA_DELEGATE_SHARED_STREAM=1 restores the single shared queue.
  static const bool shared_q = getenv("ADAPTRA_DELEGATE_SHARED_STREAM") != nullptr;
  if (shared_q) {
    ib->dstream = signal_stream(dev);
  } else if (cudaStreamCreateWithFlags(&ib->dstream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaFree(ib->mbox);
    flags_close(ib->fl);
    delete ib;
    return set_error(ADAPTRA_ECUDA, "inbox_create: stream");
  }
  ib->own_dstream = !shared_q;
  if (host_name && host_name[0]) {
    int rc = ring_open(ib->ring, host_name, n_mb, bytes, true);
    if (rc) {
      if (ib->own_dstream) cudaStreamDestroy(ib->dstream);
      cudaFree(ib->mbox);
      flags_close(ib->fl);
      delete ib;
      return rc;
    }
    ib->has_ring = true;
    Delegate::get().add(ib);
  }
  cudaDeviceSynchronize();
  *out = ib;
  return ADAPTRA_OK;
}

extern "C" int adaptra_inbox_destroy(adaptra_inbox_t ib) {
  if (!ib) return ADAPTRA_OK;
  if (ib->has_ring) {
    Delegate::get().remove(ib);
    ring_close(ib->ring);
  }
  cudaSetDevice(ib->dev);
  cudaStreamSynchronize(ib->dstream);
  if (ib->own_dstream) cudaStreamDestroy(ib->dstream);
  cudaFree(ib->mbox);
  flags_close(ib->fl);
  delete ib;
  return ADAPTRA_OK;
}

extern "C" int adaptra_inbox_export(adaptra_inbox_t ib, uint8_t* handle) {
  if (!ib || !handle) return set_error(ADAPTRA_EINVAL, "inbox_export: null");
  cudaSetDevice(ib->dev);
  cudaIpcMemHandle_t h1;
  ADAPTRA_CUDA_TRY(cudaIpcGetMemHandle(&h1, ib->mbox));
  memcpy(handle, &h1, 64);
  if (ib->fl.name.size() > 63) return set_error(ADAPTRA_ELINK, "flag segment name too long");
  memset(handle + 64, 0, 64);
  memcpy(handle + 64, ib->fl.name.c_str(), ib->fl.name.size());
  return ADAPTRA_OK;
}

extern "C" void* adaptra_inbox_slot(adaptra_inbox_t ib, int32_t mb) {
  if (!ib || mb < 0 || mb >= ib->n_mb) return nullptr;
  return (char*)ib->mbox + (size_t)mb * ib->bytes;
}

extern "C" int adaptra_recv(adaptra_inbox_t ib, int32_t mb, uint32_t epoch, void* consumer, void** slot_out) {
  if (!ib || mb < 0 || mb >= ib->n_mb) return set_error(ADAPTRA_EINVAL, "recv: bad mb");
  (void)consumer;  // ops are launched only after the wait, in the stage's stream order
  int rc = host_wait_hmem(ib->fl.h + mb, epoch);
  if (rc) return rc;
  if (slot_out) *slot_out = (char*)ib->mbox + (size_t)mb * ib->bytes;
  return ADAPTRA_OK;
}

extern "C" int adaptra_inbox_poison(adaptra_inbox_t ib) {
  if (!ib) return set_error(ADAPTRA_EINVAL, "inbox_poison: null");
  // release every waiter (abort path after a failed or timed-out iteration)
  // 0x3F3F3F3F compares >= every epoch in use (wrap-around compare)
  for (int mb = 0; mb < ib->n_mb; ++mb) __atomic_store_n((uint32_t*)(ib->fl.h + mb), 0x3F3F3F3Fu, __ATOMIC_RELEASE);
  return ADAPTRA_OK;
}

extern "C" int adaptra_inbox_reset(adaptra_inbox_t ib) {
  if (!ib) return set_error(ADAPTRA_EINVAL, "inbox_reset: null");
  cudaSetDevice(ib->dev);
  ADAPTRA_CUDA_TRY(cudaStreamSynchronize(signal_stream(ib->dev)));
  for (int mb = 0; mb < ib->n_mb; ++mb) __atomic_store_n((uint32_t*)(ib->fl.h + mb), 0u, __ATOMIC_RELEASE);
  std::fill(ib->delivered.begin(), ib->delivered.end(), 0u);
  if (ib->has_ring) memset((void*)ib->ring.flags(ib->bytes, ib->n_mb), 0, (size_t)ib->n_mb * 4);
  return ADAPTRA_OK;
}

extern "C" int adaptra_inbox_set_host(adaptra_inbox_t ib, int32_t on) {
  if (!ib) return set_error(ADAPTRA_EINVAL, "inbox_set_host: null");
  if (on && !ib->has_ring) return set_error(ADAPTRA_ELINK, "inbox has no host ring");
  ib->host_on.store(on ? 1 : 0);
  return ADAPTRA_OK;
}

// ================================================================ outbox
// Sender-side staging slots: the producing op writes here when the data does
// not go straight into the peer mailbox (P2P copy kernel, HOST path).  DIRECT
// outboxes only need them once the link fails over to the host path, so they
// are allocated then (adaptra_set_link_latency(LINK_DOWN)), not up front.
static int ensure_staging(adaptra_outbox* ob) {
  if (ob->staging) return ADAPTRA_OK;
  cudaSetDevice(ob->dev);
  if (cudaMalloc(&ob->staging, (size_t)ob->n_mb * ob->bytes) != cudaSuccess) {
    cudaGetLastError();
    ob->staging = nullptr;
    return set_error(ADAPTRA_ENOMEM, "outbox: staging cudaMalloc failed");
  }
  return ADAPTRA_OK;
}

static int outbox_common(adaptra_outbox* ob) {
  cudaSetDevice(ob->dev);
  ADAPTRA_CUDA_TRY(cudaStreamCreateWithFlags(&ob->lstream, cudaStreamNonBlocking));
  if (ob->mode == ADAPTRA_LINK_DIRECT && !remote_stores_forced()) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, ob->peer_mbox) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
      ob->remote_ce = pa.device != ob->dev;
    cudaGetLastError();
  }
  if (ob->mode != ADAPTRA_LINK_DIRECT || ob->remote_ce) {
    int rc = ensure_staging(ob);
    if (rc) return rc;
  }
  ob->ev_prod.resize(ob->n_mb);
  ob->ev_moved.resize(ob->n_mb);
  for (int k = 0; k < ob->n_mb; ++k) {
    ADAPTRA_CUDA_TRY(cudaEventCreateWithFlags(&ob->ev_prod[k], cudaEventDisableTiming));
    ADAPTRA_CUDA_TRY(cudaEventCreateWithFlags(&ob->ev_moved[k], cudaEventDisableTiming));
  }
  return ADAPTRA_OK;
}

extern "C" int adaptra_outbox_open_local(int32_t dev, adaptra_inbox_t peer, int32_t mode, adaptra_outbox_t* out) {
  if (!peer || !out || mode < 0 || mode > 2) return set_error(ADAPTRA_EINVAL, "outbox_open_local: bad args");
  auto* ob = new adaptra_outbox();
  ob->dev = dev;
  ob->n_mb = peer->n_mb;
  ob->bytes = peer->bytes;
  ob->mode = mode;
  ob->peer_mbox = (char*)peer->mbox;
  ob->peer_hflags = peer->fl.h;
  ob->peer_dflags = peer->fl.d;
  if (dev != peer->dev) {
    cudaSetDevice(dev);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer->dev, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
      delete ob;
      return set_error(ADAPTRA_ELINK, std::string("peer access: ") + cudaGetErrorString(e));
    }
    cudaGetLastError();
  }
  int rc = outbox_common(ob);
  if (!rc && peer->has_ring) {
    ob->ring = peer->ring;  // same process: share the mapping (not owner)
    ob->ring.owner = false;
    ob->ring.registered = false;
    ob->has_ring = true;
  }
  if (rc) {
    delete ob;
    return rc;
  }
  *out = ob;
  return ADAPTRA_OK;
}

extern "C" int adaptra_outbox_open_ipc(int32_t dev, const uint8_t* handle, int32_t n_mb, int64_t bytes,
                                       const char* host_name, int32_t mode, adaptra_outbox_t* out) {
  if (!handle || !out || n_mb < 1 || bytes < 16 || mode < 0 || mode > 2)
    return set_error(ADAPTRA_EINVAL, "outbox_open_ipc: bad args");
  auto* ob = new adaptra_outbox();
  ob->dev = dev;
  ob->n_mb = n_mb;
  ob->bytes = bytes;
  ob->mode = mode;
  cudaSetDevice(dev);
  cudaIpcMemHandle_t h1;
  memcpy(&h1, handle, 64);
  void* p1 = nullptr;
  cudaError_t e1 = cudaIpcOpenMemHandle(&p1, h1, cudaIpcMemLazyEnablePeerAccess);
  if (e1 != cudaSuccess) {
    delete ob;
    return set_error(ADAPTRA_ELINK, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e1));
  }
  char nm[65];
  memcpy(nm, handle + 64, 64);
  nm[64] = 0;
  int frc = flags_open(ob->fl_map, nm, n_mb, false);
  if (frc) {
    cudaIpcCloseMemHandle(p1);
    delete ob;
    return frc;
  }
  ob->peer_mbox = (char*)p1;
  ob->peer_hflags = ob->fl_map.h;
  ob->peer_dflags = ob->fl_map.d;
  ob->ipc = true;
  int rc = outbox_common(ob);
  if (!rc && host_name && host_name[0]) {
    rc = ring_open(ob->ring, host_name, n_mb, bytes, false);
    ob->has_ring = rc == ADAPTRA_OK;
  }
  if (rc) {
    delete ob;
    return rc;
  }
  *out = ob;
  return ADAPTRA_OK;
}

extern "C" int adaptra_outbox_close(adaptra_outbox_t ob) {
  if (!ob) return ADAPTRA_OK;
  cudaSetDevice(ob->dev);
  cudaStreamSynchronize(ob->lstream);
  // let the gate release every item that references this outbox
  while (ob->inflight.load() > 0) std::this_thread::sleep_for(std::chrono::microseconds(50));
  cudaStreamSynchronize(signal_stream(ob->dev));
  for (auto e : ob->ev_prod) cudaEventDestroy(e);
  for (auto e : ob->ev_moved) cudaEventDestroy(e);
  cudaStreamDestroy(ob->lstream);
  if (ob->staging) cudaFree(ob->staging);
  if (ob->ipc) {
    cudaIpcCloseMemHandle(ob->peer_mbox);
    flags_close(ob->fl_map);
  }
  if (ob->has_ring && ob->ring.registered) ring_close(ob->ring);
  delete ob;
  return ADAPTRA_OK;
}

// true when messages take the delegated host path: the link failed, or the
// policy moved a straggling link there (adaptra_link_set_path)
static bool ob_down(adaptra_outbox_t ob) {
  return ob->latency.load() == ADAPTRA_LINK_DOWN || ob->force_host.load();
}

extern "C" void* adaptra_outbox_dst(adaptra_outbox_t ob, int32_t mb) {
  if (!ob || mb < 0 || mb >= ob->n_mb) return nullptr;
  if (ob->mode == ADAPTRA_LINK_DIRECT && !ob->remote_ce && !ob_down(ob)) return ob->peer_mbox + (size_t)mb * ob->bytes;
  return (char*)ob->staging + (size_t)mb * ob->bytes;
}

extern "C" int adaptra_set_link_latency(adaptra_outbox_t ob, int64_t ns) {
  if (!ob || ns < 0) return set_error(ADAPTRA_EINVAL, "set_link_latency: bad args");
  if (ns == ADAPTRA_LINK_DOWN && !ob->has_ring) return set_error(ADAPTRA_ELINK, "link down but no host ring");
  if (ns == ADAPTRA_LINK_DOWN) {
    int rc = ensure_staging(ob);
    if (rc) return rc;
  }
  ob->latency.store(ns);
  return ADAPTRA_OK;
}

static void record_delay(adaptra_outbox_t ob, int64_t ready, int64_t rel) {
  int64_t d = rel - ready;
  ob->n_msgs.fetch_add(1);
  ob->sum_delay.fetch_add(d);
  int64_t m = ob->max_delay.load();
  while (d > m && !ob->max_delay.compare_exchange_weak(m, d)) {
  }
}

extern "C" int adaptra_send(adaptra_outbox_t ob, int32_t mb, void* producer, uint32_t epoch) {
  if (!ob || mb < 0 || mb >= ob->n_mb) return set_error(ADAPTRA_EINVAL, "send: bad mb");
  cudaSetDevice(ob->dev);
  const int64_t lat = ob->latency.load();
  const bool down = lat == ADAPTRA_LINK_DOWN;
  const int mode = (down || ob->force_host.load()) ? ADAPTRA_LINK_HOST : ob->mode;
  ADAPTRA_CUDA_TRY(cudaEventRecord(ob->ev_prod[mb], (cudaStream_t)producer));
  uint32_t* flag = ob->peer_dflags + mb;
  volatile uint32_t* hflag_peer = ob->peer_hflags + mb;
  if (mode == ADAPTRA_LINK_DIRECT || mode == ADAPTRA_LINK_P2P) {
    cudaEvent_t ready = ob->ev_prod[mb];
    const bool moved = mode == ADAPTRA_LINK_P2P || ob->remote_ce;
    if (moved) {
      ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(ob->lstream, ob->ev_prod[mb], 0));
      char* dst = ob->peer_mbox + (size_t)mb * ob->bytes;
      const char* src = (char*)ob->staging + (size_t)mb * ob->bytes;
      if (mode == ADAPTRA_LINK_P2P) {
        int rc = copy_async(dst, src, ob->bytes, ob->lstream);  // copy kernel (SM stores)
        if (rc) return rc;
      } else {
        ADAPTRA_CUDA_TRY(cudaMemcpyAsync(dst, src, ob->bytes, cudaMemcpyDeviceToDevice, ob->lstream));  // copy engine
      }
      ADAPTRA_CUDA_TRY(cudaEventRecord(ob->ev_moved[mb], ob->lstream));
      ready = ob->ev_moved[mb];
    }
    if (lat == 0) {
      // no injected latency: post the flag right behind the producer (DIRECT
      // within a GPU) or behind the copy, on the same stream (stream order
      // puts it after the data stores)
      return stream_write(moved ? ob->lstream : (cudaStream_t)producer, flag, epoch);
    }
    // injected latency: the gate thread posts the flag from the host c ns
    // after the data is in place
    ob->inflight.fetch_add(1);
    Gate::get().push(GateItem{ready, lat, [ob, hflag_peer, epoch](int64_t r, int64_t t) {
                                record_delay(ob, r, t);
                                __atomic_store_n((uint32_t*)hflag_peer, epoch, __ATOMIC_RELEASE);
                                ob->inflight.fetch_sub(1);
                              }});
    return ADAPTRA_OK;
  }
  // HOST (delegated) path: D2H into the pinned ring on the side stream, then
  // the host flag after the delegated-path latency.
  if (!ob->has_ring) return set_error(ADAPTRA_ELINK, "send: host path without a ring");
  ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(ob->lstream, ob->ev_prod[mb], 0));
  ADAPTRA_CUDA_TRY(cudaMemcpyAsync(ob->ring.data(ob->bytes, mb), (char*)ob->staging + (size_t)mb * ob->bytes,
                                   ob->bytes, cudaMemcpyDeviceToHost, ob->lstream));
  ADAPTRA_CUDA_TRY(cudaEventRecord(ob->ev_moved[mb], ob->lstream));
  volatile uint32_t* hflag = ob->ring.flags(ob->bytes, ob->n_mb) + mb;
  const int64_t hlat = down ? 0 : lat;  // a down link has no injected latency of its own
  ob->inflight.fetch_add(1);
  Gate::get().push(GateItem{ob->ev_moved[mb], hlat, [ob, hflag, epoch](int64_t r, int64_t t) {
                              record_delay(ob, r, t);
                              __atomic_store_n((uint32_t*)hflag, epoch, __ATOMIC_RELEASE);
                              ob->inflight.fetch_sub(1);
                            }});
  return ADAPTRA_OK;
}

extern "C" int adaptra_recv_blocking(adaptra_inbox_t ib, int32_t mb, uint32_t epoch, void** slot_out) {
  if (!ib || mb < 0 || mb >= ib->n_mb) return set_error(ADAPTRA_EINVAL, "recv_blocking: bad mb");
  cudaSetDevice(ib->dev);
  int rc = host_wait_hmem(ib->fl.h + mb, epoch);
  if (rc) return rc;
  if (slot_out) *slot_out = (char*)ib->mbox + (size_t)mb * ib->bytes;
  return ADAPTRA_OK;
}

extern "C" int adaptra_send_wait(adaptra_outbox_t ob, int32_t mb, uint32_t epoch) {
  if (!ob || mb < 0 || mb >= ob->n_mb) return set_error(ADAPTRA_EINVAL, "send_wait: bad mb");
  cudaSetDevice(ob->dev);
  if (ob_down(ob)) {  // delegated path: wait for the host flag
    volatile uint32_t* hf = ob->ring.flags(ob->bytes, ob->n_mb) + mb;
    while ((int32_t)(*hf - epoch) < 0) std::this_thread::sleep_for(std::chrono::microseconds(5));
    return ADAPTRA_OK;
  }
  return host_wait_hmem(ob->peer_hflags + mb, epoch);  // the receiver's flag
}

extern "C" int adaptra_link_stats(adaptra_outbox_t ob, int64_t* n, int64_t* sum, int64_t* mx) {
  if (!ob) return set_error(ADAPTRA_EINVAL, "link_stats: null");
  if (n) *n = ob->n_msgs.load();
  if (sum) *sum = ob->sum_delay.load();
  if (mx) *mx = ob->max_delay.load();
  return ADAPTRA_OK;
}

extern "C" int adaptra_link_stats_take(adaptra_outbox_t ob, int64_t* n, int64_t* sum, int64_t* mx) {
  if (!ob) return set_error(ADAPTRA_EINVAL, "link_stats_take: null");
  if (n) *n = ob->n_msgs.load();
  if (sum) *sum = ob->sum_delay.load();
  const int64_t m = ob->max_delay.exchange(0);
  if (mx) *mx = m;
  return ADAPTRA_OK;
}

namespace adaptra {
int64_t outbox_latency(adaptra_outbox_t ob) { return ob ? ob->latency.load() : 0; }
int64_t outbox_bytes(adaptra_outbox_t ob) { return ob ? ob->bytes : 0; }
void* outbox_local_slot(adaptra_outbox_t ob, int mb) {
  if (!ob || mb < 0 || mb >= ob->n_mb || ensure_staging(ob)) return nullptr;
  return (char*)ob->staging + (size_t)mb * ob->bytes;
}
}  // namespace adaptra

extern "C" int adaptra_link_set_path(adaptra_outbox_t ob, int32_t path) {
  if (!ob || (path != ADAPTRA_PATH_GPU && path != ADAPTRA_PATH_HOST)) return set_error(ADAPTRA_EINVAL, "link_set_path: bad args");
  if (path == ADAPTRA_PATH_HOST) {
    if (!ob->has_ring) return set_error(ADAPTRA_ELINK, "link_set_path: no host ring");
    int rc = ensure_staging(ob);
    if (rc) return rc;
  }
  ob->force_host.store(path == ADAPTRA_PATH_HOST ? 1 : 0);
  return ADAPTRA_OK;
}
