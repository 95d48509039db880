// txb_halo.cuh — the peer-memory window layout and the system-scope
// spin / release primitives of the halo exchange (txb_halo.cu: put /
// assemble; protocol described there), kept apart from the kernels so other
// kernels can take part in the protocol.
#pragma once

#include <cstdint>
#include <cstdlib>

namespace txb {
namespace halo {

constexpr int MAX_RANKS = 64;

struct WindowHeader {
  unsigned long long flags[MAX_RANKS];
  unsigned long long acks[MAX_RANKS];
  unsigned int counters[4];  // [0..1] put, [2..3] assemble, by epoch parity
  int error;                 // 0 ok, 1 put timed out waiting for an ack, 2 assemble timed out waiting for a
                             // flag, 3 a sender published a poisoned flag (its put failed)
  unsigned int put_failed[2];  // by epoch parity: some CTA of this rank's put skipped its stores
  int pad;
};

// A flag published by a put that failed carries this bit: the receiver sees
// the epoch arrive, but knows the rows are not there (error 3) instead of
// assembling a stale slot.
constexpr unsigned long long POISON = 1ull << 63;
constexpr int64_t HEADER_BYTES = 2048;
static_assert(sizeof(WindowHeader) <= HEADER_BYTES, "window header");

__device__ __forceinline__ unsigned long long load_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void store_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *p >= want (acquire, system scope); false on timeout.
__device__ __forceinline__ bool wait_at_least(const unsigned long long* p, unsigned long long want,
                                              unsigned long long timeout_ns) {
  const unsigned long long t0 = now_ns();
  while (load_acquire_sys(p) < want) {
    if (now_ns() - t0 > timeout_ns) return false;
    __nanosleep(200);
  }
  return true;
}

// Spin until the flag's epoch (poison bit masked) reaches `want`; returns the
// flag value seen, or 0 on timeout.
__device__ __forceinline__ unsigned long long wait_flag(const unsigned long long* p, unsigned long long want,
                                                        unsigned long long timeout_ns) {
  const unsigned long long t0 = now_ns();
  unsigned long long v;
  while (((v = load_acquire_sys(p)) & ~POISON) < want) {
    if (now_ns() - t0 > timeout_ns) return 0;
    __nanosleep(200);
  }
  return v;
}

__host__ __device__ __forceinline__ WindowHeader* header(void* w) { return reinterpret_cast<WindowHeader*>(w); }

inline unsigned long long timeout_ns() {
  const char* v = std::getenv("TXB_HALO_TIMEOUT_MS");
  const long long ms = v && *v ? std::atoll(v) : 10000;
  return (unsigned long long)(ms > 1 ? ms : 1) * 1000000ull;
}

}  // namespace halo
}  // namespace txb
