#include <initializer_list>
#include <cstdint>
#include <cstdio>
#include <chrono>
extern "C" int alora_hash_chains(int32_t, const uint8_t* const*, const uint32_t* const*, const int64_t*, int32_t, const char* const*, const int64_t* const*, uint8_t* const*, int32_t);
int main(){ static uint32_t t[12][2048]; static int64_t off[129]={0}; static uint8_t out[12][2048];
 const uint32_t* tp[12]; const char* kb[12]; const int64_t* ko[12]; uint8_t* op[12]; int64_t nb[12];
 for(int c=0;c<12;c++){for(int i=0;i<2048;i++)t[c][i]=i*7+c; tp[c]=t[c]; kb[c]=""; ko[c]=off; op[c]=out[c]; nb[c]=128;}
 for(int th: {1,2,4,8}){
 for(int i=0;i<20;i++) alora_hash_chains(12,nullptr,tp,nb,16,kb,ko,op,th);
 auto a=std::chrono::steady_clock::now(); for(int i=0;i<200;i++) alora_hash_chains(12,nullptr,tp,nb,16,kb,ko,op,th);
 auto b=std::chrono::steady_clock::now(); printf("threads %d: %.1f us/call\n", th, std::chrono::duration<double,std::micro>(b-a).count()/200);}}
