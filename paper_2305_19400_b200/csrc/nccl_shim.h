// nccl_shim.h -- minimal NCCL interface: point-to-point for the slab halo
// exchange (a5), AllGather for the band-partition partials.  NCCL is resolved at run time with dlopen (the copy PyTorch
// ships and has usually already loaded), so libbte.so has no link-time NCCL
// dependency and single-GPU use never touches it.
#pragma once
#include <cstddef>
#include <string>

#include <cuda_runtime.h>

int nccl_shim_init(void **comm, const void *unique_id_128b, int nranks, int rank, std::string *err);
int nccl_shim_send(void *comm, const double *buf, size_t count, int peer, cudaStream_t s, std::string *err);
int nccl_shim_recv(void *comm, double *buf, size_t count, int peer, cudaStream_t s, std::string *err);
// in-place when send == recv + rank*count (band-partition partials)
int nccl_shim_allgather(void *comm, const double *send, double *recv, size_t count, cudaStream_t s,
                        std::string *err);
// the communicator's own view: ncclCommCount / ncclCommUserRank
int nccl_shim_comm_info(void *comm, int *nranks, int *rank, std::string *err);
int nccl_shim_group_start(std::string *err);
int nccl_shim_group_end(std::string *err);
void nccl_shim_destroy(void *comm);
