#include <execinfo.h>
#include <signal.h>
#include <unistd.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static void h(int sig){ void* b[64]; int n=backtrace(b,64); backtrace_symbols_fd(b,n,2);
 FILE* f=fopen("/proc/self/maps","r"); char line[512]; while(f&&fgets(line,512,f)) if(strstr(line,".so")&&strstr(line,"r-xp")) fputs(line,stderr); _exit(139);}
#include <string.h>
__attribute__((constructor)) static void init(void){ signal(SIGSEGV,h); }
