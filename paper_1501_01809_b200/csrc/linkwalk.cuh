// linkwalk.cuh -- host helper of the link / star tile planners (ltile.cu, thtile.cu).
#pragma once
#include <algorithm>
#include <utility>
#include <vector>

namespace loam_gpu {

// The link of a mesh edge (tetrahedra) or of a vertex (triangles): every cell
// around it contributes the segment (P, Q) of its two other vertices.  A manifold edge's segments form
// one closed ring (interior) or one open fan (boundary).  Writes the vertex
// sequence p_0 .. p_n (cell i = (v, w, p_i, p_{i+1}); a ring repeats p_0 at the
// end) as coordinate ids; false when the segments are anything else.
struct LinkWalk {
  static constexpr int kMax = 64;
  int nid[kMax], nx[kMax], deg[kMax], nb[kMax][2], nn = 0;
  bool seen[kMax];
  int find(int node, int x) {
    for (int i = 0; i < nn; ++i)
      if (nid[i] == node) return i;
    if (nn == kMax) return -1;
    nid[nn] = node;
    nx[nn] = x;
    deg[nn] = 0;
    return nn++;
  }
  bool add(int P, int xp, int Q, int xq) {
    const int a = find(P, xp), b = find(Q, xq);
    if (a < 0 || b < 0 || a == b || deg[a] == 2 || deg[b] == 2) return false;
    nb[a][deg[a]++] = b;
    nb[b][deg[b]++] = a;
    return true;
  }
  bool walk(int ncell, std::vector<int>& seq) {
    int ends = 0, start = 0;
    for (int i = nn - 1; i >= 0; --i)
      if (deg[i] == 1) {
        ++ends;
        start = i;
      }
    const bool ring = ends == 0;
    if (ring ? (nn != ncell || nn < 3) : (ends != 2 || nn != ncell + 1)) return false;
    for (int i = 0; i < nn; ++i) seen[i] = false;
    seq.clear();
    int prev = -1, cur = start;
    seq.push_back(nx[cur]);
    seen[cur] = true;
    for (int k = 0; k < ncell; ++k) {
      int nxt;
      if (prev < 0) nxt = nb[cur][0];
      else {
        if (deg[cur] != 2) return false;
        nxt = nb[cur][0] == prev ? nb[cur][1] : nb[cur][0];
      }
      if (k + 1 < ncell || !ring) {
        if (seen[nxt]) return false; // a second component, or a doubled segment
        seen[nxt] = true;
      } else if (nxt != start) return false;
      seq.push_back(nx[nxt]);
      prev = cur;
      cur = nxt;
    }
    return ring ? true : deg[cur] == 1;
  }
};


// even-aligned, gap-merged id runs of a tile's vertex window (as the other tile packers)
inline int link_runs(std::vector<int>& ids, int limit, std::vector<std::pair<int, int>>& rr) {
  constexpr int kGap = 8;
  std::sort(ids.begin(), ids.end());
  rr.clear();
  int slots = 0;
  for (int v : ids) {
    const int lo = v & ~1, hi = std::min(limit, (v + 2) & ~1);
    if (!rr.empty() && lo <= rr.back().second + kGap) rr.back().second = std::max(rr.back().second, hi);
    else rr.emplace_back(lo, hi);
  }
  for (auto& x : rr) slots += x.second - x.first;
  return slots;
}

} // namespace loam_gpu
