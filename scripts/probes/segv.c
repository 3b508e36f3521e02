#define _GNU_SOURCE
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>
#include <pthread.h>
static void h(int sig) {
  void *b[64]; int n = backtrace(b, 64);
  char msg[128]; int l = snprintf(msg, sizeof msg, "SIGNAL %d in thread %lu\n", sig, (unsigned long)pthread_self());
  write(2, msg, l);
  backtrace_symbols_fd(b, n, 2);
  _exit(139);
}
__attribute__((constructor)) static void init(void) { signal(SIGSEGV, h); signal(SIGABRT, h); }
