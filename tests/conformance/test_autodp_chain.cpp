// The one reference autodp case the conformance run skips
// ("the full 8-4-2-1 transition chain keeps every invariant",
// proj/tests/test_autodp.cpp:71-95) inserts a range whose begin() and end()
// come from two different temporaries (UB: it loops forever with either
// library).  Same invariants, restated with one materialised vector, run
// against libeps_b200.so:
//   * every K in the chain 8 -> 4 -> 2 -> 1 on 2x8 validates;
//   * R = 16 / K and the message group is all 16 ranks;
//   * each newly activated rank receives exactly one message, ranks that
//     were already active receive none.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <map>
#include <set>
#include <vector>

#include "eps/autodp.hpp"

using namespace eps;

TEST_CASE("8-4-2-1 transition chain on 2x8 (restated without the range UB)") {
  ClusterSpec c;
  c.node_count = 2;
  c.gpus_per_node = 8;
  Topology topo(c, 8);
  const std::vector<int> first = topo.active_ranks();
  std::set<int> active(first.begin(), first.end());
  for (int new_k : {4, 2, 1}) {
    const TransitionResult res = transition(topo, new_k, {});
    CHECK_NOTHROW(res.topology.validate());
    CHECK(res.topology.replica_width() == 16 / new_k);
    CHECK(res.topology.message_group().size() == 16);
    std::map<int, int> received;
    for (const TransitionMessage& m : res.messages) received[m.receiver]++;
    const std::vector<int> now = res.topology.active_ranks();
    CHECK(now.size() == static_cast<size_t>(16 / new_k));
    for (int rank : now) {
      if (active.count(rank)) CHECK(received.count(rank) == 0);
      else CHECK(received[rank] == 1);
    }
    active.insert(now.begin(), now.end());
    topo = res.topology;
  }
}
