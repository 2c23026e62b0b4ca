// The `fastleg` command-line tool built on the B200 library: subcommands
// dlt / idlt / ndct / leg2cheb / nodes / compare / bench (include/fastleg/cli.hpp).
//   g++ -std=c++20 -O2 -Iinclude tools/fastleg_b200.cpp -Lpaper_1505_00354_b200 -lfastleg_b200
#include "fastleg/cli.hpp"

int main(int argc, char** argv) { return fastleg::cli::run(argc, argv); }
