// profiler.cu -- optional per-kernel CUDA-event timing of the library's own launches, used
// by bench.py to report the dominant kernel's live duration inside the timed region.
// Off by default; when on, one event is recorded on the launching stream after every
// kernel (and at API entry), and kernel i's time is elapsed(event i-1, event i).
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "../../include/sla_b200.h"
#include "common.cuh"

namespace slab {

namespace {
struct Rec {
  std::string name;
  cudaEvent_t ev;
};
struct Prof {
  bool on = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::pair<double, long long>> acc;  // ms, launches
};
Prof& prof() {
  static Prof p;
  return p;
}
cudaEvent_t take_event() {
  Prof& p = prof();
  if (!p.pool.empty()) {
    cudaEvent_t e = p.pool.back();
    p.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void flush() {
  Prof& p = prof();
  if (p.recs.empty()) return;
  cudaEventSynchronize(p.recs.back().ev);
  for (size_t i = 1; i < p.recs.size(); ++i) {
    if (p.recs[i].name.empty()) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.recs[i - 1].ev, p.recs[i].ev);
    auto& a = p.acc[p.recs[i].name];
    a.first += ms;
    a.second += 1;
  }
  for (auto& r : p.recs) p.pool.push_back(r.ev);
  p.recs.clear();
}
}  // namespace

bool prof_enabled() { return prof().on; }

void prof_mark(const char* name, cudaStream_t st) {
  Prof& p = prof();
  if (!p.on) return;
  cudaEvent_t e = take_event();
  cudaEventRecord(e, st);
  p.recs.push_back({name ? name : "", e});
  if (p.recs.size() > 4096) flush();
}

}  // namespace slab

extern "C" {

// enable: 1 on, 0 off (clears).  report: "name ms launches\n" lines, returns bytes needed.
int sla_b200_profiler(int enable) {
  slab::Prof& p = slab::prof();
  slab::flush();
  p.on = enable != 0;
  p.acc.clear();
  return 0;
}

size_t sla_b200_profiler_report(char* buf, size_t len) {
  slab::flush();
  std::string out;
  char line[256];
  for (auto& [name, a] : slab::prof().acc) {
    std::snprintf(line, sizeof line, "%s %.6f %lld\n", name.c_str(), a.first, a.second);
    out += line;
  }
  if (buf && len) {
    std::snprintf(buf, len, "%s", out.c_str());
  }
  return out.size() + 1;
}

}  // extern "C"
