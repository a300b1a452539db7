// Peer-memory halo exchange for the z-slab runtime (SURVEY.md §8 row a26, §5 "step 2";
// reference runtime.py:323-342 exchange_halos).
//
// Every rank exposes an inbox in its own device memory -- two parity slots x (lo, hi)
// boundary planes plus one flag word per slot -- and maps its neighbours' inboxes
// into its address space (CUDA IPC; over NVLink when the neighbour is another GPU of
// the node).  Iteration k writes its first / last plane straight into the lower /
// upper neighbour's slot k % 2 (a stream-ordered peer copy), then k_halo_signal
// publishes k + 1 in that slot's flag after a system-scope fence.  Before the kernel
// that reads the halos, k_halo_wait spins on its own flags until both neighbours have
// published k + 1.  No NCCL call and no host round trip are on the data path; the
// per-iteration scalar allreduce keeps the ranks in lockstep, which makes two parity
// slots sufficient (slot k % 2 is rewritten at k + 2, after every reader of it has
// contributed to the allreduce of k + 1).
#include "tf_common.cuh"

namespace tf {

__global__ void k_halo_signal(unsigned long long* flag, unsigned long long value) {
  __threadfence_system();  // the plane copied before this kernel is visible first
  *reinterpret_cast<volatile unsigned long long*>(flag) = value;
  __threadfence_system();
}

__global__ void k_halo_wait(const unsigned long long* flag_lo, const unsigned long long* flag_hi,
                            unsigned long long value) {
  const volatile unsigned long long* lo = flag_lo;
  const volatile unsigned long long* hi = flag_hi;
  while ((lo && *lo < value) || (hi && *hi < value)) __nanosleep(200);
  __threadfence_system();  // acquire: the halo planes are read after this
}

int halo_signal(unsigned long long* flag, unsigned long long value, cudaStream_t st) {
  k_halo_signal<<<1, 1, 0, st>>>(flag, value);
  return check_launch("k_halo_signal");
}

int halo_wait(const unsigned long long* flag_lo, const unsigned long long* flag_hi,
              unsigned long long value, cudaStream_t st) {
  k_halo_wait<<<1, 1, 0, st>>>(flag_lo, flag_hi, value);
  return check_launch("k_halo_wait");
}

}  // namespace tf
