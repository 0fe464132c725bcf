// Peer-memory transport: block buffers are read by their consumers straight
// out of the producing GPU's memory over NVLink (CUDA IPC mappings of a
// symmetric buffer region), so a transport round of the schedule
// (inc/fabric.hpp:95-106 -- one Fabric::deliver per block) costs one
// readiness flag instead of a copy: the merge or assembly that consumes a
// block reads it remotely, overlapping the transfer with its own work.
//
// Protocol, per iteration e (a device-resident counter, so CUDA-graph replays
// see fresh values):
//   k_begin    e = ++epoch; wait until every peer finished iteration e-1
//              (peers may still read our block buffers until then)
//   publish    the select producing a block, as soon as its cluster is done:
//              fence, then store e into each consumer's flag for the block
//              (remote store; peer_publish, common.cuh)
//   wait       the merge, single-block select or assembly consuming a remote
//              block: spin (acquire, system scope) until its local flag
//              reaches e (peer_wait, common.cuh)
//   k_publish  after the last remote read of the iteration: store e into
//              every peer's done[rank] flag
// Waits are bounded (10 s, SPARDL_PEER_TIMEOUT_MS): a peer that never arrives
// sets *err, every later wait of the iteration returns at once, the writers
// of persistent state (residual finalize, ledger, controller) skip their
// stores, and the next sync() reports the error and poisons the context
// until reset_state().
#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

__global__ void k_begin(long long* epoch, const long long* const* done, int n, int32_t* err,
                        unsigned long long timeout_ns) {
  pdl_enter();
  __shared__ long long e;
  if (threadIdx.x == 0) {
    e = *epoch + 1;
    *epoch = e;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) spin_until(done[i], e - 1, err, timeout_ns);
}

__global__ void k_publish(long long* const* targets, int n, const long long* epoch) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long e = *epoch;
  __threadfence_system();
  st_release_sys(targets[i], e);
}


}  // namespace

namespace {
thread_local cudaError_t g_launch_error = cudaSuccess;
}
void note_launch(cudaError_t e) {
  if (e != cudaSuccess && g_launch_error == cudaSuccess) g_launch_error = e;
}
cudaError_t take_launch_error() {
  const cudaError_t e = g_launch_error;
  g_launch_error = cudaSuccess;
  return e;
}

int launch_begin(long long* epoch, const long long* const* done, int n, int32_t* err,
                 unsigned long long timeout_ns, cudaStream_t s) {
  launch_pdl(k_begin, dim3(1), dim3(32), 0, s, epoch, done, n, err, timeout_ns);
  return 1;
}

int launch_publish(long long* const* targets, int n, const long long* epoch, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_pdl(k_publish, dim3((n + 127) / 128), dim3(128), 0, s, targets, n, epoch);
  return 1;
}


}  // namespace sdl
