// Host sampling profiler for the launch-bound workloads (DGNN_HOST_SAMPLE=<us>):
// SIGPROF every <us> microseconds of process CPU time records the calling
// frames (backtrace); at exit the functions most often on the stack (leaf
// and inclusive) are printed to stderr with their share of the samples.
// Diagnostic only — no effect unless the variable is set.
#include <cxxabi.h>
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <sys/time.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace dgnn {
namespace {

constexpr int kDepth = 24;
constexpr int kMaxSamples = 100000;
void* g_frames[kMaxSamples][kDepth];
int g_depth[kMaxSamples];
std::atomic<int> g_n{0};

void on_prof(int) {
  const int i = g_n.fetch_add(1, std::memory_order_relaxed);
  if (i >= kMaxSamples) return;
  g_depth[i] = backtrace(g_frames[i], kDepth);
}

std::string name_of(void* pc) {
  Dl_info info;
  if (dladdr(pc, &info) && info.dli_sname) {
    int st = 0;
    char* dem = abi::__cxa_demangle(info.dli_sname, nullptr, nullptr, &st);
    std::string s = st == 0 && dem ? dem : info.dli_sname;
    std::free(dem);
    if (s.size() > 110) s = s.substr(0, 110);
    return s;
  }
  if (dladdr(pc, &info) && info.dli_fname) return std::string("[") + info.dli_fname + "]";
  return "?";
}

void report() {
  const int n = std::min(g_n.load(), kMaxSamples);
  if (n == 0) return;
  std::map<std::string, int> leaf, incl;
  for (int i = 0; i < n; ++i) {
    if (g_depth[i] <= 2) continue;
    leaf[name_of(g_frames[i][2])]++;  // frames 0-1: the handler and the signal trampoline
    std::vector<std::string> seen;
    for (int k = 2; k < g_depth[i]; ++k) {
      std::string s = name_of(g_frames[i][k]);
      if (std::find(seen.begin(), seen.end(), s) == seen.end()) {
        seen.push_back(s);
        incl[s]++;
      }
    }
  }
  auto dump = [&](const char* title, const std::map<std::string, int>& m) {
    std::vector<std::pair<int, std::string>> v;
    for (const auto& [k, c] : m) v.push_back({c, k});
    std::sort(v.rbegin(), v.rend());
    std::fprintf(stderr, "[dgnn host sample] %s (%d samples)\n", title, n);
    for (size_t i = 0; i < v.size() && i < 40; ++i)
      std::fprintf(stderr, "  %5.1f%%  %s\n", 100.0 * v[i].first / n, v[i].second.c_str());
  };
  dump("leaf", leaf);
  dump("inclusive", incl);
}

struct Init {
  Init() {
    const char* e = std::getenv("DGNN_HOST_SAMPLE");
    if (!e) return;
    const long us = std::max(100L, std::atol(e));
    struct sigaction sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.sa_handler = on_prof;
    sa.sa_flags = SA_RESTART;
    sigaction(SIGPROF, &sa, nullptr);
    itimerval tv;
    tv.it_interval.tv_sec = us / 1000000;
    tv.it_interval.tv_usec = us % 1000000;
    tv.it_value = tv.it_interval;
    setitimer(ITIMER_PROF, &tv, nullptr);
    std::atexit(report);
  }
} g_init;

}  // namespace
}  // namespace dgnn
