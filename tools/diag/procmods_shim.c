// LD_PRELOAD shim (diagnosis only): fopen("/proc/modules") -> /dev/null when
// the sandbox's procfs has no /proc/modules (libcufile reads it with a
// getline loop that waits for EOF and never sees one when the open failed).
#define _GNU_SOURCE
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>
#include <unistd.h>

static const char* fix(const char* p) {
  return (p && !strcmp(p, "/proc/modules") && access(p, R_OK)) ? "/dev/null" : p;
}
FILE* fopen(const char* p, const char* m) {
  static FILE* (*real)(const char*, const char*);
  if (!real) real = (FILE * (*)(const char*, const char*)) dlsym(RTLD_NEXT, "fopen");
  return real(fix(p), m);
}
FILE* fopen64(const char* p, const char* m) {
  static FILE* (*real)(const char*, const char*);
  if (!real) real = (FILE * (*)(const char*, const char*)) dlsym(RTLD_NEXT, "fopen64");
  return real(fix(p), m);
}
