// Error reporting and launch accounting shared by every translation unit of libatom.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

namespace atom {

unsigned long long g_launch_count = 0;
static thread_local char g_err[1024];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

}  // namespace atom
