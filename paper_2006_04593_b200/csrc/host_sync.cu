// Host-side scheduling words of the in-process two-party runtime
// (runtime.run_local_pair; the reference runs the two parties as two Python
// threads over queues, runtime.py:285-311).
//
// Both party programs are Python, so only one of them runs at a time (the GIL).
// With blocking queues every hand-over between the parties -- a party waiting
// for the peer's frame, the peer taking the interpreter, a worker picking up a
// job -- is a futex sleep and a kernel wake-up, tens of microseconds each,
// during which the GPU has nothing queued (the online round cannot launch its
// evaluation before both masked messages exist). Here a waiting party instead
// spins in native code with the GIL released (ctypes drops it for the call) on
// 64-bit words: a frame counter per inbox and a `turn` word naming the party
// that may run Python next. The running party passes the turn when it blocks
// or finishes, so the interpreter is handed over in well under a microsecond
// and is never contended. The turn is advisory: a waiter whose condition holds
// runs anyway `grace_s` after it became true, so a party that blocks inside
// some other call while holding the turn cannot deadlock the pair.
// A hand-over (pass the turn, post a counter) and the wait that follows it are
// ONE call: were they two, the thread released by the hand-over would find the
// GIL still held between the calls and sleep on it.
#include <cuda_runtime.h>
#include <sched.h>
#include <stdint.h>
#include <time.h>

#include "../../include/ariann_fss.h"
#include "common.cuh"

namespace {

inline double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#elif defined(__aarch64__)
    asm volatile("yield" ::: "memory");
#endif
}

inline int64_t load_acq(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }

}  // namespace

extern "C" {

int64_t fss_host_load(const int64_t* word) { return word ? load_acq(word) : 0; }

void fss_host_store(int64_t* word, int64_t value) {
    if (word) __atomic_store_n(word, value, __ATOMIC_RELEASE);
}

int64_t fss_host_add(int64_t* word, int64_t delta) {
    return word ? __atomic_add_fetch(word, delta, __ATOMIC_ACQ_REL) : 0;
}

int fss_host_wait(const int64_t* word, int64_t target, int64_t* turn, int64_t me, int64_t pass_to,
                  int64_t* bump, double spin_s, double grace_s, double timeout_s) {
    if (!word) return FSS_EINVAL;
    // The caller's last writes before it starts waiting happen here, after
    // ctypes dropped the GIL: whoever they release finds the GIL free.
    if (bump) __atomic_add_fetch(bump, 1, __ATOMIC_ACQ_REL);
    if (turn && pass_to >= 0) __atomic_store_n(turn, pass_to, __ATOMIC_RELEASE);
    const bool check_turn = turn && me >= 0;
    const double t0 = now_s();
    double ready_at = -1.0;  // when *word >= target was first seen
    long sleep_ns = 1000;
    bool slow = false;       // past the tight-spin phase
    for (uint64_t it = 0;; it++) {
        if (load_acq(word) >= target) {
            if (!check_turn || load_acq(turn) == me) return 0;
            // condition met, turn pending: the peer is about to hand over --
            // tight spin (no naps) for at most grace_s
            const double t = now_s();
            if (ready_at < 0) ready_at = t;
            else if (t - ready_at >= grace_s) return 0;
            cpu_relax();
            continue;
        }
        if (slow || (it & 63) == 0) {
            const double el = now_s() - t0;
            if (el >= timeout_s) return 1;
            if (el >= spin_s) {
                slow = true;
                if (el < 2 * spin_s) {
                    sched_yield();
                } else {
                    timespec ts = {0, sleep_ns};
                    nanosleep(&ts, nullptr);
                    if (sleep_ns < 50000) sleep_ns *= 2;
                }
                continue;
            }
        }
        cpu_relax();
    }
}

// Stream ordering of the party streams without torch's per-call Event objects
// (run_local_pair forks the two party streams from the caller's stream and
// joins them back; LocalTransport orders a frame's payload on the receiver's
// stream after the sender's). Events are created without timing.

int fss_event_create(void** ev) {
    if (!ev) return fssb::set_error(FSS_EINVAL, "fss_event_create: NULL out pointer");
    const cudaError_t err = cudaEventCreateWithFlags((cudaEvent_t*)ev, cudaEventDisableTiming);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_event_destroy(void* ev) {
    if (!ev) return FSS_OK;
    const cudaError_t err = cudaEventDestroy((cudaEvent_t)ev);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_event_record(void* ev, void* stream) {
    if (!ev) return fssb::set_error(FSS_EINVAL, "fss_event_record: NULL event");
    const cudaError_t err = cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

int fss_stream_wait_event(void* stream, void* ev) {
    if (!ev) return fssb::set_error(FSS_EINVAL, "fss_stream_wait_event: NULL event");
    const cudaError_t err = cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    return FSS_OK;
}

// Waiters w[0..nw) wait for the work queued so far on producers p[0..np)
// (streams of the current device; a 0 handle is the legacy default stream).
// One event per calling thread and device, re-recorded per producer: a wait
// takes the record current at the time of the wait, so the reuse is exact.
int fss_streams_link(void* waiter0, void* waiter1, int n_waiters, void* producer0, void* producer1,
                     int n_producers) {
    static thread_local cudaEvent_t evs[64] = {};
    if (n_waiters < 0 || n_waiters > 2 || n_producers < 0 || n_producers > 2)
        return fssb::set_error(FSS_EINVAL, "fss_streams_link: at most two waiters and two producers");
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    if (dev < 0 || dev >= 64) return fssb::set_error(FSS_EINVAL, "fss_streams_link: device index >= 64");
    if (!evs[dev]) {
        err = cudaEventCreateWithFlags(&evs[dev], cudaEventDisableTiming);
        if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    }
    void* const producers[2] = {producer0, producer1};
    void* const waiters[2] = {waiter0, waiter1};
    for (int i = 0; i < n_producers; i++) {
        err = cudaEventRecord(evs[dev], (cudaStream_t)producers[i]);
        if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
        for (int j = 0; j < n_waiters; j++) {
            err = cudaStreamWaitEvent((cudaStream_t)waiters[j], evs[dev], 0);
            if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
        }
    }
    return FSS_OK;
}

}  // extern "C"
