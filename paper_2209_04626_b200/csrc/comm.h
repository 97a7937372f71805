// comm.h -- NCCL transport of the sharded Jacobi engine:
// one process per GPU, ncclSend/ncclRecv of column blocks between
// neighbouring ranks after every round, ncclBroadcast / point-to-point
// gather of the working matrices at stage boundaries, and a max/sum
// all-reduce of the sweep's convergence counters.  NCCL is loaded with
// dlopen on first use (libnccl.so.2: the copy torch already mapped, or the
// system one), so the library loads and runs single-GPU without it.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace mpj {

class Comm {
public:
    int rank = 0, world = 1;
    bool active() const { return comm_ != nullptr; }
    // id: 128 bytes from nccl_unique_id() on rank 0, distributed by the caller
    int init(int rank, int world, const unsigned char* id);   // 0 or MPJSVD_ERR_*
    void destroy();
    int bcast(void* buf, size_t bytes, int root, cudaStream_t st);
    int group_start();
    int group_end();
    int send(const void* buf, size_t bytes, int peer, cudaStream_t st);
    int recv(void* buf, size_t bytes, int peer, cudaStream_t st);
    int allreduce_max_f64(double* buf, size_t count, cudaStream_t st);
    int allreduce_max_i64(long long* buf, size_t count, cudaStream_t st);
    int allreduce_sum_i32(int* buf, size_t count, cudaStream_t st);
    int async_error();   // ncclCommGetAsyncError, polled at the per-sweep synchronisation

private:
    void* comm_ = nullptr;   // ncclComm_t
};

int nccl_unique_id(unsigned char* out128);
const char* nccl_last_error();

}  // namespace mpj
