// nccl_shim.cpp -- dlopen-based NCCL binding (see nccl_shim.h).
#include "nccl_shim.h"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace {
struct Nccl {
  void *h = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGroupStart) gstart = nullptr;
  decltype(&ncclGroupEnd) gend = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  decltype(&ncclCommCount) count = nullptr;
  decltype(&ncclCommUserRank) userrank = nullptr;
};

Nccl &lib(std::string *err) {
  static Nccl n;
  static bool failed = false;  // a missing libnccl is looked up once (loopback-only runs)
  static std::mutex mu;        // loopback ranks are threads: one resolver at a time
  std::lock_guard<std::mutex> lk(mu);
  if (n.h) return n;
  if (failed) {
    if (err) *err = "cannot dlopen libnccl.so.2 (import torch first or set BTE_NCCL_LIB)";
    return n;
  }
  const char *cands[] = {getenv("BTE_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  for (const char *c : cands) {
    if (!c) continue;
    n.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (n.h) break;
  }
  if (!n.h) {
    failed = true;
    if (err) *err = "cannot dlopen libnccl.so.2 (import torch first or set BTE_NCCL_LIB)";
    return n;
  }
  n.init = (decltype(n.init))dlsym(n.h, "ncclCommInitRank");
  n.send = (decltype(n.send))dlsym(n.h, "ncclSend");
  n.recv = (decltype(n.recv))dlsym(n.h, "ncclRecv");
  n.allgather = (decltype(n.allgather))dlsym(n.h, "ncclAllGather");
  n.gstart = (decltype(n.gstart))dlsym(n.h, "ncclGroupStart");
  n.gend = (decltype(n.gend))dlsym(n.h, "ncclGroupEnd");
  n.destroy = (decltype(n.destroy))dlsym(n.h, "ncclCommDestroy");
  n.errstr = (decltype(n.errstr))dlsym(n.h, "ncclGetErrorString");
  n.count = (decltype(n.count))dlsym(n.h, "ncclCommCount");
  n.userrank = (decltype(n.userrank))dlsym(n.h, "ncclCommUserRank");
  if (!n.init || !n.send || !n.recv || !n.allgather || !n.gstart || !n.gend || !n.destroy || !n.errstr || !n.count ||
      !n.userrank) {
    if (err) *err = "libnccl is missing symbols (send/recv/allgather/group)";
    dlclose(n.h);
    n.h = nullptr;
  }
  return n;
}

int check(ncclResult_t r, std::string *err) {
  if (r == ncclSuccess) return 0;
  if (err) *err = lib(nullptr).errstr ? lib(nullptr).errstr(r) : "nccl error";
  return 1;
}
}  // namespace

// ---------------------------------------------------------------- in-process loopback transport
// A unique id that starts with "BTELOOP" selects an in-process stand-in for
// NCCL: the ranks are threads of one process (one device, or several), every
// send/recv/AllGather of a group is matched across the ranks at group end and
// executed as device copies in stream order -- the receiver's stream waits for
// the sender's data (an event recorded when the send was posted), copies, and
// records a "done" event the sender's stream waits on before it may touch the
// buffer again, as with NCCL.  So the library's own multi-rank code -- plans,
// send/recv buffers, pack/scatter kernels, comm stream, overlap events, the
// all-gathered energy -- runs unchanged on one GPU; only the wire is replaced.
// No kernel waits on another rank (the host rendezvous does), so nothing can
// hang the device.  Test infrastructure (tests/test_gpu_loopback.py).
namespace loopback {
constexpr uint32_t kMagic = 0x504f4f4cu;  // tag of a loopback communicator
enum { OP_SEND = 0, OP_RECV = 1, OP_GATHER = 2 };

struct Op {
  int kind;
  const double *src;  // send buffer / gather contribution
  double *dst;        // recv buffer / gather result
  size_t count;
  int peer;
  cudaStream_t s;
  cudaEvent_t post = nullptr;               // data (send) / buffer (recv) ready in stream order
  std::vector<cudaEvent_t> done;            // consumers' completion (sender waits on these)
};

struct World {
  int nranks = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;          // barrier arrivals in the current phase
  uint64_t phase = 0;     // barrier generation
  std::vector<std::vector<Op>> posted;  // [rank] ops of the current group
  bool failed = false;
  std::string why;
};

struct Comm {
  uint32_t magic = kMagic;
  World *w = nullptr;
  int rank = 0;
};

std::mutex g_mu;
std::map<std::string, World *> g_worlds;

struct Pending {
  Comm *c;
  Op op;
};
thread_local std::vector<Pending> t_pending;
thread_local int t_depth = 0;

bool is_loop(void *comm) { return comm && static_cast<Comm *>(comm)->magic == kMagic; }

// all ranks arrive; the last one runs `last` under the lock; false on timeout
template <class F>
bool barrier(World &w, F last, std::string *err) {
  std::unique_lock<std::mutex> lk(w.mu);
  const uint64_t ph = w.phase;
  if (++w.count == w.nranks) {
    last();
    w.count = 0;
    ++w.phase;
    w.cv.notify_all();
    return true;
  }
  if (!w.cv.wait_for(lk, std::chrono::seconds(120), [&] { return w.phase != ph; })) {
    w.failed = true;
    w.why = "loopback: a peer rank did not reach the exchange within 120 s";
    if (err) *err = w.why;
    return false;
  }
  return !w.failed;
}

int ck(cudaError_t e, std::string *err) {
  if (e == cudaSuccess) return 0;
  if (err) *err = std::string("loopback: ") + cudaGetErrorString(e);
  return 1;
}

int run_group(Comm *c, std::vector<Op> ops, std::string *err) {
  World &w = *c->w;
  const int r = c->rank;
  for (Op &o : ops) {  // stream-ordered readiness of each buffer
    if (ck(cudaEventCreateWithFlags(&o.post, cudaEventDisableTiming), err)) return 1;
    if (ck(cudaEventRecord(o.post, o.s), err)) return 1;
  }
  {
    std::lock_guard<std::mutex> lk(w.mu);
    w.posted[r] = std::move(ops);
  }
  if (!barrier(w, [] {}, err)) return 1;
  // receiver side: copy from the matching send (k-th recv from p <-> k-th send to r)
  std::vector<Op> &mine = w.posted[r];
  std::map<int, int> nth;
  for (Op &o : mine) {
    if (o.kind == OP_RECV) {
      const int k = nth[o.peer]++;
      Op *snd = nullptr;
      int seen = 0;
      for (Op &q : w.posted[o.peer])
        if (q.kind == OP_SEND && q.peer == r && seen++ == k) {
          snd = &q;
          break;
        }
      if (!snd || snd->count != o.count) {
        if (err) *err = "loopback: unmatched send/recv (rank " + std::to_string(r) + " <- " + std::to_string(o.peer) + ")";
        return 1;
      }
      cudaEvent_t d;
      if (ck(cudaStreamWaitEvent(o.s, snd->post, 0), err) ||
          ck(cudaMemcpyAsync(o.dst, snd->src, o.count * sizeof(double), cudaMemcpyDefault, o.s), err) ||
          ck(cudaEventCreateWithFlags(&d, cudaEventDisableTiming), err) || ck(cudaEventRecord(d, o.s), err))
        return 1;
      std::lock_guard<std::mutex> lk(w.mu);
      snd->done.push_back(d);
    } else if (o.kind == OP_GATHER) {
      for (int p = 0; p < w.nranks; ++p) {
        Op *g = nullptr;
        for (Op &q : w.posted[p])
          if (q.kind == OP_GATHER) {
            g = &q;
            break;
          }
        if (!g || g->count != o.count) {
          if (err) *err = "loopback: AllGather not posted by every rank with one count";
          return 1;
        }
        double *to = o.dst + (size_t)p * o.count;
        if (p == r && g->src == to) continue;  // in place
        cudaEvent_t d;
        if ((p != r && ck(cudaStreamWaitEvent(o.s, g->post, 0), err)) ||
            ck(cudaMemcpyAsync(to, g->src, o.count * sizeof(double), cudaMemcpyDefault, o.s), err) ||
            ck(cudaEventCreateWithFlags(&d, cudaEventDisableTiming), err) || ck(cudaEventRecord(d, o.s), err))
          return 1;
        std::lock_guard<std::mutex> lk(w.mu);
        g->done.push_back(d);
      }
    }
  }
  if (!barrier(w, [] {}, err)) return 1;
  // sender side: the buffer is free once every consumer's copy is done
  for (Op &o : mine) {
    for (cudaEvent_t d : o.done)
      if (ck(cudaStreamWaitEvent(o.s, d, 0), err)) return 1;
  }
  return barrier(w, [&w] {
    for (auto &v : w.posted) {
      for (Op &o : v) {
        cudaEventDestroy(o.post);
        for (cudaEvent_t d : o.done) cudaEventDestroy(d);
      }
      v.clear();
    }
  }, err) ? 0 : 1;
}

int post(void *comm, const Op &op, std::string *err) {
  Comm *c = static_cast<Comm *>(comm);
  if (t_depth > 0) {
    t_pending.push_back({c, op});
    return 0;
  }
  return run_group(c, {op}, err);
}

int init(void **comm, const void *uid, int nranks, int rank, std::string *err) {
  const std::string key(static_cast<const char *>(uid), 128);
  World *w;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_worlds.find(key);
    if (it == g_worlds.end()) {
      w = new World;
      w->nranks = nranks;
      w->posted.resize(nranks);
      g_worlds[key] = w;
    } else {
      w = it->second;
    }
    if (w->nranks != nranks || rank < 0 || rank >= nranks) {
      if (err) *err = "loopback: inconsistent nranks/rank";
      return 1;
    }
    ++w->refs;
  }
  Comm *c = new Comm;
  c->w = w;
  c->rank = rank;
  *comm = c;
  return 0;
}

void destroy(Comm *c) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (--c->w->refs == 0) {
    for (auto it = g_worlds.begin(); it != g_worlds.end(); ++it)
      if (it->second == c->w) {
        g_worlds.erase(it);
        break;
      }
    delete c->w;
  }
  delete c;
}
}  // namespace loopback

int nccl_shim_init(void **comm, const void *uid, int nranks, int rank, std::string *err) {
  if (std::memcmp(uid, "BTELOOP", 7) == 0) return loopback::init(comm, uid, nranks, rank, err);
  Nccl &n = lib(err);
  if (!n.h) return 1;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  ncclComm_t c = nullptr;
  if (check(n.init(&c, nranks, id, rank), err)) return 1;
  *comm = c;
  return 0;
}

int nccl_shim_send(void *comm, const double *buf, size_t count, int peer, cudaStream_t s, std::string *err) {
  if (loopback::is_loop(comm)) return loopback::post(comm, {loopback::OP_SEND, buf, nullptr, count, peer, s}, err);
  return check(lib(err).send(buf, count, ncclFloat64, peer, (ncclComm_t)comm, s), err);
}

int nccl_shim_recv(void *comm, double *buf, size_t count, int peer, cudaStream_t s, std::string *err) {
  if (loopback::is_loop(comm)) return loopback::post(comm, {loopback::OP_RECV, nullptr, buf, count, peer, s}, err);
  return check(lib(err).recv(buf, count, ncclFloat64, peer, (ncclComm_t)comm, s), err);
}

int nccl_shim_allgather(void *comm, const double *send, double *recv, size_t count, cudaStream_t s,
                        std::string *err) {
  if (loopback::is_loop(comm)) return loopback::post(comm, {loopback::OP_GATHER, send, recv, count, -1, s}, err);
  return check(lib(err).allgather(send, recv, count, ncclFloat64, (ncclComm_t)comm, s), err);
}

int nccl_shim_comm_info(void *comm, int *nranks, int *rank, std::string *err) {
  if (loopback::is_loop(comm)) {
    *nranks = static_cast<loopback::Comm *>(comm)->w->nranks;
    *rank = static_cast<loopback::Comm *>(comm)->rank;
    return 0;
  }
  Nccl &n = lib(err);
  if (!n.h) return 1;
  if (check(n.count((ncclComm_t)comm, nranks), err)) return 1;
  return check(n.userrank((ncclComm_t)comm, rank), err);
}

// Group calls open/close a loopback group on this thread too; a thread's
// group holds the operations of one communicator (the library's usage).
int nccl_shim_group_start(std::string *err) {
  ++loopback::t_depth;
  Nccl &n = lib(nullptr);
  if (n.h) return check(n.gstart(), err);
  return 0;  // no libnccl: loopback only
}
int nccl_shim_group_end(std::string *err) {
  int rc = 0;
  Nccl &n = lib(nullptr);
  if (n.h) rc = check(n.gend(), err);
  if (--loopback::t_depth == 0 && !loopback::t_pending.empty()) {
    std::vector<loopback::Pending> pend;
    pend.swap(loopback::t_pending);
    std::vector<loopback::Op> ops;
    for (auto &p : pend) {
      if (p.c != pend[0].c) {  // one communicator per group (the library's usage)
        if (err) *err = "loopback: a group mixes communicators";
        return 1;
      }
      ops.push_back(p.op);
    }
    if (loopback::run_group(pend[0].c, std::move(ops), err)) rc = 1;
  }
  return rc;
}

void nccl_shim_destroy(void *comm) {
  if (loopback::is_loop(comm)) return loopback::destroy(static_cast<loopback::Comm *>(comm));
  Nccl &n = lib(nullptr);
  if (n.h && comm) n.destroy((ncclComm_t)comm);
}
