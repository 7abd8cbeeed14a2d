// Sample the user-space instruction pointer of one thread (ptrace attach,
// GETREGS, detach) N times and print it with the mapping it falls in — a
// poor man's profiler for a spinning library call (no gdb/perf in the image).
//   rip_sample <tid> <pid> [n]
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/ptrace.h>
#include <sys/user.h>
#include <sys/wait.h>
#include <unistd.h>

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  pid_t tid = atoi(argv[1]);
  int pid = atoi(argv[2]);
  int n = argc > 3 ? atoi(argv[3]) : 10;
  char mp[64];
  snprintf(mp, sizeof mp, "/proc/%d/maps", pid);
  for (int i = 0; i < n; ++i) {
    if (ptrace(PTRACE_ATTACH, tid, 0, 0)) { perror("attach"); return 1; }
    waitpid(tid, 0, __WALL);
    struct user_regs_struct r;
    ptrace(PTRACE_GETREGS, tid, 0, &r);
    unsigned long rip = r.rip;
    ptrace(PTRACE_DETACH, tid, 0, 0);
    FILE* f = fopen(mp, "r");
    char line[512], hit[512] = "?";
    unsigned long lo = 0, hi = 0, off = 0, base = 0;
    while (f && fgets(line, sizeof line, f)) {
      unsigned long a, b, o;
      char perm[8];
      if (sscanf(line, "%lx-%lx %7s %lx", &a, &b, perm, &o) == 4 && rip >= a && rip < b) {
        lo = a; hi = b; off = o; base = a;
        strncpy(hit, line, sizeof hit - 1);
      }
    }
    if (f) fclose(f);
    printf("rip=%lx file_off=%lx %s", rip, rip - base + off, hit);
    usleep(200000);
  }
  return 0;
}
