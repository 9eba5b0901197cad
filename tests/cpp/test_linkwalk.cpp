// CPU test of the planners' host helper (csrc/linkwalk.cuh): the link of a
// mesh edge (tetrahedra) or vertex (triangles) as one ring or one fan, and the
// even-aligned, gap-merged window runs.  No GPU needed.
#include <cstdio>
#include <vector>

#include "linkwalk.cuh"

using loam_gpu::LinkWalk;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                            \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(c)) {                                                             \
      ++g_fail;                                                             \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);          \
    }                                                                       \
  } while (0)

static bool walk(const std::vector<std::pair<int, int>>& segs, std::vector<int>& seq) {
  LinkWalk lw;
  for (auto& s : segs)
    if (!lw.add(s.first, 10 * s.first, s.second, 10 * s.second)) return false; // x = 10 * node: the walk reports x
  return lw.walk((int)segs.size(), seq);
}

int main() {
  std::vector<int> seq;
  // a ring of five cells, segments in scrambled order and orientation: closed, every vertex once, p_0 repeated
  CHECK(walk({{3, 4}, {1, 0}, {2, 3}, {0, 4}, {1, 2}}, seq));
  CHECK(seq.size() == 6 && seq.front() == seq.back());
  {
    std::vector<int> seen(5, 0);
    for (size_t i = 0; i + 1 < seq.size(); ++i) {
      CHECK(seq[i] % 10 == 0 && seq[i] / 10 < 5);
      ++seen[seq[i] / 10];
      const int a = seq[i] / 10, b = seq[i + 1] / 10; // consecutive entries are a segment of the input
      CHECK((a + 1) % 5 == b || (b + 1) % 5 == a);
    }
    for (int c : seen) CHECK(c == 1);
  }
  // a fan of three cells (boundary edge): open, starts and ends at the two degree-1 vertices
  CHECK(walk({{7, 8}, {6, 7}, {8, 9}}, seq));
  CHECK(seq.size() == 4 && seq.front() != seq.back());
  CHECK((seq.front() == 60 && seq.back() == 90) || (seq.front() == 90 && seq.back() == 60));
  // a single cell is a fan of one segment
  CHECK(walk({{1, 2}}, seq) && seq.size() == 2);
  // not a link of a manifold edge: two components, a branching vertex, a doubled segment, a 2-ring
  CHECK(!walk({{0, 1}, {1, 2}, {2, 0}, {5, 6}}, seq));
  CHECK(!walk({{0, 1}, {1, 2}, {1, 3}}, seq));
  CHECK(!walk({{0, 1}, {0, 1}}, seq));
  CHECK(!walk({{0, 1}, {1, 2}, {2, 0}, {3, 4}, {4, 5}, {5, 3}}, seq));
  CHECK(!walk({{0, 0}}, seq)); // degenerate segment
  // window runs: even-aligned, merged across gaps of at most 8 ids, clipped to the limit
  {
    std::vector<int> ids{21, 5, 4, 40, 13, 99};
    std::vector<std::pair<int, int>> rr;
    const int slots = loam_gpu::link_runs(ids, 100, rr);
    CHECK(rr.size() == 3);
    CHECK(rr[0] == std::make_pair(4, 22));  // 4..5, 13, 21 chained by gaps <= 8 (6 -> 12, 14 -> 20)
    CHECK(rr[1] == std::make_pair(40, 42));
    CHECK(rr[2] == std::make_pair(98, 100)); // clipped at the vertex count
    CHECK(slots == 18 + 2 + 2);
    for (auto& r : rr) CHECK(r.first % 2 == 0);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
