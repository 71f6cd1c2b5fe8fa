// Host unit test of the sharded wait policy (paper_1902_09465_b200/csrc/host_wait.h):
// ready / device error / peer error / timeout, with a simulated clock and event.
#include <cstdio>
#include <cstdlib>

#include "host_wait.h"

using namespace aknn;

static int check(bool ok, const char *what) {
  if (!ok) std::printf("FAIL %s\n", what);
  return ok ? 0 : 1;
}

int main() {
  int bad = 0;
  {  // ready after 1000 polls, no error: no abort
    int polls = 0, aborts = 0;
    double t = 0;
    WaitResult r = wait_loop([&] { return ++polls > 1000 ? 1 : 0; }, [] { return false; }, [&] { ++aborts; },
                             [&] { return t += 0.001; }, 50.0);
    bad += check(r == WAIT_READY && aborts == 0 && polls == 1001, "ready");
  }
  {  // device error is reported without touching the communicator
    int aborts = 0;
    WaitResult r = wait_loop([] { return -1; }, [] { return true; }, [&] { ++aborts; }, [] { return 0.0; }, 1.0);
    bad += check(r == WAIT_DEVICE_ERROR && aborts == 0, "device error");
  }
  {  // peer error after some polls: abort exactly once
    int polls = 0, aborts = 0;
    WaitResult r = wait_loop([&] { ++polls; return 0; }, [&] { return polls > 5000; }, [&] { ++aborts; },
                             [] { return 0.0; }, 0.0);
    bad += check(r == WAIT_PEER_ERROR && aborts == 1, "peer error");
  }
  {  // a dead peer: the event never completes, no error is reported -> the deadline
    int aborts = 0;
    double t = 0;
    WaitResult r = wait_loop([] { return 0; }, [] { return false; }, [&] { ++aborts; },
                             [&] { return t += 1.0; }, 10000.0);
    bad += check(r == WAIT_TIMEOUT && aborts == 1 && t > 10000.0 && t < 10100.0, "timeout");
  }
  {  // timeout 0 = no deadline: completes late without an abort
    int polls = 0, aborts = 0;
    double t = 0;
    WaitResult r = wait_loop([&] { return ++polls > 2000000 ? 1 : 0; }, [] { return false; }, [&] { ++aborts; },
                             [&] { return t += 100.0; }, 0.0);
    bad += check(r == WAIT_READY && aborts == 0, "no deadline");
  }
  std::printf(bad ? "wait_test: %d failures\n" : "wait_test: ok\n", bad);
  return bad ? 1 : 0;
}
