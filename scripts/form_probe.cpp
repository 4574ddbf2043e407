#include <chrono>
#include <cstdio>
#include <vector>
#include "taskfuse_b200.h"
static volatile long long completed = 0;
static long long published = 0, seen = 0;
int busy(void*, int32_t) { if (published != seen) { seen = published; return 1; } return completed < published; }
int main() {
  for (int A : {1, 4, 16, 64, 128}) {
    tf_region* r; int P = 4096 / A; if (P < 1) P = 1;
    tf_region_create("reconstruct", A, P, 1, &r);
    std::vector<int64_t> buf(8192);
    double best = 1e9;
    for (int rep = 0; rep < 50; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      long long teams = 0;
      for (int i = 0; i < 4096; ++i) {
        if (tf_region_watch_count(r, 0) > 0 && !busy(nullptr, 0)) {
          int k = tf_region_stream_idle(r, 0, buf.data(), 8192);
          for (int j = 0; j < k; ++j) { published += tf_region_team_size(r, buf[j]); tf_region_release_team(r, buf[j]); teams++; }
        }
        tf_enter_result res;
        tf_region_enter(r, i, busy, nullptr, &res);
        if (res.closed != 0) { published += tf_region_team_size(r, res.team); tf_region_release_team(r, res.team); teams++; }
      }
      int k = tf_region_stream_idle(r, 0, buf.data(), 8192);
      for (int j = 0; j < k; ++j) { tf_region_release_team(r, buf[j]); }
      auto t1 = std::chrono::steady_clock::now();
      double us = std::chrono::duration<double, std::micro>(t1 - t0).count();
      if (us < best) best = us;
    }
    printf("A=%d: best %.1f us per 4096 arrivals\n", A, best);
    tf_region_destroy(r);
  }
}
