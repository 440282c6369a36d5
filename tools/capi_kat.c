#include <stdio.h>
#include <dlfcn.h>
#include <stddef.h>
#include <stdlib.h>
typedef int (*conv_t)(int, const size_t*, const double*, const size_t*, const double*, double*);
int main() {
  int argc_ = 0; (void)argc_; extern char** environ; const char* path = getenv("NDC_LIB") ? getenv("NDC_LIB") : "./paper_1711_11224_b200/libndconv_b200.so"; void* h = dlopen(path, RTLD_NOW);
  if (!h) { printf("dlopen: %s\n", dlerror()); return 1; }
  conv_t f = (conv_t)dlsym(h, "ndc_conv_full_f64");
  const char* (*err)(void) = (const char* (*)(void))dlsym(h, "ndc_last_error");
  size_t xe[1] = {2}, ke[1] = {3}; double x[2] = {1, 2}, k[3] = {1, 1, 1}, y[4];
  int rc = f(1, xe, x, ke, k, y);
  printf("rc=%d %s y=%g %g %g %g\n", rc, err(), y[0], y[1], y[2], y[3]);
  return 0;
}
