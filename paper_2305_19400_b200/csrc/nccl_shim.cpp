// nccl_shim.cpp -- dlopen-based NCCL binding (see nccl_shim.h).
#include "nccl_shim.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>

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
  if (n.h) return n;
  const char *cands[] = {getenv("BTE_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  for (const char *c : cands) {
    if (!c) continue;
    n.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (n.h) break;
  }
  if (!n.h) {
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

int nccl_shim_init(void **comm, const void *uid, int nranks, int rank, std::string *err) {
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
  return check(lib(err).send(buf, count, ncclFloat64, peer, (ncclComm_t)comm, s), err);
}

int nccl_shim_recv(void *comm, double *buf, size_t count, int peer, cudaStream_t s, std::string *err) {
  return check(lib(err).recv(buf, count, ncclFloat64, peer, (ncclComm_t)comm, s), err);
}

int nccl_shim_allgather(void *comm, const double *send, double *recv, size_t count, cudaStream_t s,
                        std::string *err) {
  return check(lib(err).allgather(send, recv, count, ncclFloat64, (ncclComm_t)comm, s), err);
}

int nccl_shim_comm_info(void *comm, int *nranks, int *rank, std::string *err) {
  Nccl &n = lib(err);
  if (!n.h) return 1;
  if (check(n.count((ncclComm_t)comm, nranks), err)) return 1;
  return check(n.userrank((ncclComm_t)comm, rank), err);
}

int nccl_shim_group_start(std::string *err) { return check(lib(err).gstart(), err); }
int nccl_shim_group_end(std::string *err) { return check(lib(err).gend(), err); }

void nccl_shim_destroy(void *comm) {
  Nccl &n = lib(nullptr);
  if (n.h && comm) n.destroy((ncclComm_t)comm);
}
