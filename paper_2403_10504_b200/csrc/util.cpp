// Error reporting and launch accounting shared by every translation unit of libatom.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

namespace atom {

unsigned long long g_launch_count = 0;

// launches per kernel family since load (tests check which kernels a step actually ran)
static std::mutex g_log_mu;
static std::map<std::string, unsigned long long>& launch_log() {
  static std::map<std::string, unsigned long long> m;
  return m;
}
void count_launch_named(const char* name) {
  std::lock_guard<std::mutex> lk(g_log_mu);
  ++launch_log()[name];
}
std::string launch_log_text() {
  std::lock_guard<std::mutex> lk(g_log_mu);
  std::string out;
  char buf[160];
  for (auto& kv : launch_log()) {
    snprintf(buf, sizeof buf, "%s %llu\n", kv.first.c_str(), kv.second);
    out += buf;
  }
  return out;
}
static thread_local char g_err[1024];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

}  // namespace atom
