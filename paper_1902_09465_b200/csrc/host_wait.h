// host_wait.h -- the host-side wait policy of the sharded round loop (pure host logic,
// no CUDA / NCCL types, so it is unit-tested on CPUs: tests/cpin/wait_test.cpp).
//
// A rank waits for its stream by polling an event (see capi.cu sync_spin); in a
// point-sharded query (one process per GPU, one ncclAllGather per round) a dead or
// failing peer would leave that event pending forever.  While polling, the waiter also
// polls the communicator's asynchronous error state and a wall-clock deadline; on a
// peer error or a timeout it aborts the communicator (so the pending collective and
// every other rank's matching one complete with an error instead of hanging) and
// reports AKNN_ENCCL.
#pragma once

namespace aknn {

enum WaitResult { WAIT_READY = 0, WAIT_DEVICE_ERROR = 1, WAIT_PEER_ERROR = 2, WAIT_TIMEOUT = 3 };

// ready():     1 done, 0 pending, -1 device / runtime error
// peer_err():  true when the communicator reports an asynchronous error
// abort():     aborts the communicator (called at most once)
// now_ms():    a monotonic clock in milliseconds
// timeout_ms:  <= 0 waits forever (peer errors are still detected)
template <class Ready, class PeerErr, class Abort, class Clock>
WaitResult wait_loop(Ready &&ready, PeerErr &&peer_err, Abort &&abort, Clock &&now_ms, double timeout_ms,
                     unsigned poll_every = 256) {
  const double t0 = now_ms();
  for (unsigned it = 0;; ++it) {
    const int r = ready();
    if (r > 0) return WAIT_READY;
    if (r < 0) return WAIT_DEVICE_ERROR;
    // the communicator and the clock are polled every `poll_every` event queries
    if (it % poll_every != 0) continue;
    if (peer_err()) {
      abort();
      return WAIT_PEER_ERROR;
    }
    if (timeout_ms > 0.0 && now_ms() - t0 > timeout_ms) {
      abort();
      return WAIT_TIMEOUT;
    }
  }
}

}  // namespace aknn
